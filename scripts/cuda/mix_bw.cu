// HBM ceiling for a densify-shaped traffic mix: per 16-B chunk read, R 16-B
// chunks written (R = 5 ~ cfg1 densify: 66 MB read / 328 MB written per batch),
// streaming, grid-stride, 4 independent loads in flight per thread; plus the
// same written through 80 KB shared-memory tiles with 1-D TMA bulk stores (the
// densify store path).  Reports GB/s of (read + write) bytes, best of 5.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mix_bw mix_bw.cu
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int R>
__global__ void mix(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n_in) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_in; i += stride) {
        uint4 v = in[i];
#pragma unroll
        for (int r = 0; r < R; ++r) out[i * R + r] = make_uint4(v.x + r, v.y, v.z, v.w);
    }
}

// coalesced 1:R: thread i reads in[i], writes out[i + r * n_in] (R coalesced write streams)
template <int R>
__global__ void mix_coal(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n_in) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_in; i += stride) {
        uint4 v = in[i];
#pragma unroll
        for (int r = 0; r < R; ++r) out[i + r * n_in] = make_uint4(v.x + r, v.y, v.z, v.w);
    }
}

// smem tile like tile_store, but streamed out by all threads with STG.128
__global__ void __launch_bounds__(256) tile_stg(const uint4* __restrict__ in, size_t n_in, char* __restrict__ out,
                                                size_t tiles, unsigned tile_bytes) {
    extern __shared__ __align__(128) uint4 tile[];
    unsigned acc = 0;
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const size_t per = tile_bytes / 16 / 5;
        for (size_t i = threadIdx.x; i < per; i += blockDim.x) acc += in[(t * per + i) % n_in].x;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < tile_bytes / 16; i += blockDim.x) tile[i] = make_uint4(acc, i, 0, 0);
        __syncthreads();
        uint4* o = reinterpret_cast<uint4*>(out + t * tile_bytes);
        for (unsigned i = threadIdx.x; i < tile_bytes / 16; i += blockDim.x) o[i] = tile[i];
    }
}

// each CTA: read its share of `in` (sum to keep the loads), fill an 80 KB smem tile, bulk-store it
__global__ void __launch_bounds__(256) tile_store(const uint4* __restrict__ in, size_t n_in, char* __restrict__ out,
                                                  size_t tiles, unsigned tile_bytes) {
    extern __shared__ __align__(128) uint4 tile[];
    unsigned acc = 0;
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        // read this tile's share of the input (1/5 of the tile bytes)
        const size_t per = tile_bytes / 16 / 5;
        for (size_t i = threadIdx.x; i < per; i += blockDim.x) acc += in[(t * per + i) % n_in].x;
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        for (unsigned i = threadIdx.x; i < tile_bytes / 16; i += blockDim.x) tile[i] = make_uint4(acc, i, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * tile_bytes),
                         "r"(static_cast<unsigned>(__cvta_generic_to_shared(tile))), "r"(tile_bytes) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t out_bytes = 328ull << 20, in_bytes = out_bytes / 5;
    uint4 *in, *out;
    CK(cudaMalloc(&in, in_bytes));
    CK(cudaMalloc(&out, out_bytes * 4));
    CK(cudaMemset(in, 1, in_bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int reps = 20;
    auto bench = [&](auto launch, const char* name, double bytes) {
        float best = 1e30f;
        for (int k = 0; k < 5; ++k) {
            cudaEventRecord(e0);
            for (int r = 0; r < reps; ++r) launch(r);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        std::printf("{\"kernel\": \"%s\", \"GBps\": %.1f}\n", name, bytes * reps / (best / 1e3) / 1e9);
    };
    const size_t n_in = in_bytes / 16;
    // rotate over 4 output buffers so consecutive launches do not hit L2
    bench([&](int r) { mix<5><<<sms * 8, 256>>>(in, out + (r % 4) * (out_bytes / 16), n_in); }, "stg 1:5 read:write",
          double(in_bytes + out_bytes));
    bench([&](int r) { mix<1><<<sms * 8, 256>>>(in, out + (r % 4) * (out_bytes / 16), n_in); }, "stg 1:1 copy",
          double(2 * in_bytes));
    bench([&](int r) { mix_coal<5><<<sms * 8, 256>>>(in, out + (r % 4) * (out_bytes / 16), n_in); },
          "stg coalesced 1:5", double(in_bytes + out_bytes));
    const unsigned tb = 80 * 1024;
    CK(cudaFuncSetAttribute(tile_stg, cudaFuncAttributeMaxDynamicSharedMemorySize, tb));
    bench([&](int r) { tile_stg<<<sms * 2, 256, tb>>>(in, n_in, reinterpret_cast<char*>(out) + (r % 4) * out_bytes, out_bytes / tb, tb); },
          "stg 80KB tiles 1:5", double(in_bytes + out_bytes));
    CK(cudaFuncSetAttribute(tile_store, cudaFuncAttributeMaxDynamicSharedMemorySize, tb));
    const size_t tiles = out_bytes / tb;
    bench([&](int r) { tile_store<<<sms * 2, 256, tb>>>(in, n_in, reinterpret_cast<char*>(out) + (r % 4) * out_bytes, tiles, tb); },
          "tma 80KB tiles 1:5", double(in_bytes + out_bytes));
    return 0;
}
