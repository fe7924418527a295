// HBM ceiling for a densify-shaped traffic mix: per 16-B chunk read, R 16-B
// chunks written (R = 5 ~ cfg1 densify: 66 MB read / 328 MB written per batch),
// streaming, grid-stride, 4 independent loads in flight per thread; plus the
// same written through 80 KB shared-memory tiles with 1-D TMA bulk stores (the
// densify store path).  Reports GB/s of (read + write) bytes, best of 5.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mix_bw mix_bw.cu
#include <cuda.h>
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

// write-only ceilings (K4o writes 16 B per byte it reads): STG.128 grid-stride, and
// shared tiles of tile_bytes written by 1-D TMA bulk stores (two tiles alternating)
__global__ void fill_stg(uint4* __restrict__ out, size_t n) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = make_uint4(unsigned(i), 1, 2, 3);
}
__global__ void __launch_bounds__(256) fill_tma(char* __restrict__ out, size_t tiles, unsigned tile_bytes) {
    extern __shared__ __align__(128) uint4 tile[];
    unsigned it = 0;
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        uint4* tb = tile + (it & 1u) * (tile_bytes / 16);
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        for (unsigned i = threadIdx.x; i < tile_bytes / 16; i += blockDim.x) tb[i] = make_uint4(unsigned(t), i, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * tile_bytes),
                         "r"(static_cast<unsigned>(__cvta_generic_to_shared(tb))), "r"(tile_bytes) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// tile_store with an L2 evict_first policy on the bulk stores (output lines leave L2 first)
__global__ void __launch_bounds__(256) tile_store_ef(const uint4* __restrict__ in, size_t n_in, char* __restrict__ out,
                                                     size_t tiles, unsigned tile_bytes) {
    extern __shared__ __align__(128) uint4 tile[];
    unsigned acc = 0;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const size_t per = tile_bytes / 16 / 5;
        for (size_t i = threadIdx.x; i < per; i += blockDim.x) acc += in[(t * per + i) % n_in].x;
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        for (unsigned i = threadIdx.x; i < tile_bytes / 16; i += blockDim.x) tile[i] = make_uint4(acc, i, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                         ::"l"(out + t * tile_bytes), "r"(static_cast<unsigned>(__cvta_generic_to_shared(tile))),
                         "r"(tile_bytes), "l"(pol) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the [b, n_var] f32 output written by 2-D tensor-map TMA stores (cp.async.bulk.tensor.2d):
// box = 256 columns x BR rows (BR*1 KB of smem), tiles clipped at the n_var edge by the TMA unit
__global__ void __launch_bounds__(256) tile_tensor2d(const uint4* __restrict__ in, size_t n_in,
                                                     const __grid_constant__ CUtensorMap tm, unsigned rows,
                                                     unsigned cols, unsigned br) {
    extern __shared__ __align__(128) uint4 tile[];
    const unsigned ct = (cols + 255) / 256, rt = rows / br, tiles = ct * rt, tile_bytes = br * 1024;
    unsigned acc = 0;
    for (unsigned t = blockIdx.x; t < tiles; t += gridDim.x) {
        const size_t per = tile_bytes / 16 / 5;
        for (size_t i = threadIdx.x; i < per; i += blockDim.x) acc += in[(size_t(t) * per + i) % n_in].x;
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        for (unsigned i = threadIdx.x; i < tile_bytes / 16; i += blockDim.x) tile[i] = make_uint4(acc, i, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const int c0 = static_cast<int>((t % ct) * 256), r0 = static_cast<int>((t / ct) * br);
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                         ::"l"(&tm), "r"(c0), "r"(r0), "r"(static_cast<unsigned>(__cvta_generic_to_shared(tile)))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

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
    CK(cudaFuncSetAttribute(tile_store_ef, cudaFuncAttributeMaxDynamicSharedMemorySize, tb));
    bench([&](int r) { tile_store_ef<<<sms * 2, 256, tb>>>(in, n_in, reinterpret_cast<char*>(out) + (r % 4) * out_bytes, tiles, tb); },
          "tma 80KB tiles 1:5 L2 evict_first", double(in_bytes + out_bytes));
    // write-only (out_bytes per launch, rotating over 4 buffers)
    bench([&](int r) { fill_stg<<<sms * 8, 256>>>(out + (r % 4) * (out_bytes / 16), out_bytes / 16); },
          "stg write-only", double(out_bytes));
    for (unsigned wb : {4096u, 16384u, 40960u}) {
        CK(cudaFuncSetAttribute(fill_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * wb));
        const int per_sm = wb <= 4096 ? 8 : wb <= 16384 ? 6 : 2;
        char name[96];
        std::snprintf(name, sizeof name, "tma %u KB tiles write-only", wb / 1024);
        bench([&](int r) { fill_tma<<<sms * per_sm, 256, 2 * wb>>>(reinterpret_cast<char*>(out) + (r % 4) * out_bytes,
                                                                  out_bytes / wb, wb); },
              name, double(out_bytes));
    }
    // 2-D tensor-map stores into a [rows, 20000] f32 matrix (cfg1's dense batch shape)
    EncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
    const unsigned cols = 20000, rows = static_cast<unsigned>(out_bytes / (cols * 4));
    for (unsigned br : {32u, 64u, 80u}) {
        const unsigned rws = rows / br * br;
        CUtensorMap tm[4];
        for (int k = 0; k < 4; ++k) {
            const cuuint64_t dims[2] = {cols, rws}, strides[1] = {cols * 4ull};
            const cuuint32_t box[2] = {256, br}, es[2] = {1, 1};
            if (enc(&tm[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, reinterpret_cast<char*>(out) + k * out_bytes, dims,
                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                std::printf("tensor map encode failed\n");
                return 1;
            }
        }
        const unsigned sm_bytes = br * 1024;
        CK(cudaFuncSetAttribute(tile_tensor2d, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
        const int per_sm = br <= 64 ? 3 : 2;
        char name[96];
        std::snprintf(name, sizeof name, "tma tensor 2d 256 cols x %u rows, %d CTAs/SM, 1:5", br, per_sm);
        bench([&](int r) { tile_tensor2d<<<sms * per_sm, 256, sm_bytes>>>(in, n_in, tm[r % 4], rws, cols, br); }, name,
              double(in_bytes) + double(rws) * cols * 4);
    }
    return 0;
}
