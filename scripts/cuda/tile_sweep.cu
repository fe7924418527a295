// Write-heavy HBM ceiling for densify-shaped kernels, swept over the tile shape:
// each CTA reads 1/R of a tile's bytes (R = 0: no reads), fills a shared-memory
// tile and writes it with ONE 1-D TMA bulk store (densify's store path); NB
// tile buffers per CTA (NB = 2: the next tile is filled while the previous
// store drains).  Output rotates over 4 buffers of 590 MB (cfg2's batch), so
// launches miss L2.  Prints GB/s of (read + write), best of 5 x 20 launches.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tile_sweep tile_sweep.cu
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void __launch_bounds__(256) tile_store(const uint4* __restrict__ in, size_t n_in, char* __restrict__ out,
                                                  size_t tiles, unsigned tile_bytes, unsigned ratio, unsigned nb) {
    extern __shared__ __align__(128) uint4 smem[];
    unsigned acc = 0, k = 0;
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
        uint4* tile = smem + (k % nb) * (tile_bytes / 16);
        if (ratio) {
            const size_t per = tile_bytes / 16 / ratio;
            for (size_t i = threadIdx.x; i < per; i += blockDim.x) acc += in[(t * per + i) % n_in].x;
        }
        if (threadIdx.x == 0) {
            if (nb == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
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
    if (acc == 0xdeadbeef) out[0] = 1;
}

int main() {
    const size_t out_bytes = 590ull << 20, in_bytes = out_bytes / 5;
    uint4 *in;
    char* out;
    CK(cudaMalloc(&in, in_bytes));
    CK(cudaMalloc(&out, out_bytes * 4));
    CK(cudaMemset(in, 1, in_bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaFuncSetAttribute(tile_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const size_t n_in = in_bytes / 16;
    const unsigned ratios[] = {5, 20, 0};
    const unsigned tiles_kb[] = {16, 24, 32, 40, 48, 64, 80, 100};
    for (unsigned R : ratios)
        for (unsigned nb : {1u, 2u})
            for (unsigned tk : tiles_kb) {
                const unsigned tb = tk * 1024, smem = tb * nb;
                if (smem > 220 * 1024) continue;
                int occ = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tile_store, 256, smem));
                const size_t tiles = out_bytes / tb;
                const double bytes = double(tiles) * tb + (R ? double(tiles) * (tb / 16 / R) * 16 : 0.0);
                float best = 1e30f;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaEventRecord(e0);
                    for (int r = 0; r < 20; ++r)
                        tile_store<<<sms * occ, 256, smem>>>(in, n_in, out + (r % 4) * out_bytes, tiles, tb, R, nb);
                    cudaEventRecord(e1);
                    CK(cudaEventSynchronize(e1));
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                std::printf("{\"read_ratio\": %u, \"buffers\": %u, \"tile_kb\": %u, \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", R,
                            nb, tk, occ, bytes * 20 / (best / 1e3) / 1e9);
            }
    return 0;
}
