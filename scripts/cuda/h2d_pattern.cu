// PCIe H2D calibration for the loader's staging pattern: per step, 64 copies of
// ~1 MB blocks from random offsets of a pinned host image (cfg1: f = 64 rows of
// ~16 KB), as (a) 64 cudaMemcpyAsync, (b) one cudaMemcpyBatchAsync, (c) two
// streams, against (d) one contiguous copy of the same bytes.
// Build: nvcc -O2 -o h2d_pattern h2d_pattern.cu ; run on the B200 box.
#include <cuda_runtime.h>

#include <cstdio>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
    const size_t img = 1600ull << 20, blk = 1u << 20, nb = 64, steps = 40;
    void* h = nullptr;
    void* d = nullptr;
    CK(cudaHostAlloc(&h, img, cudaHostAllocDefault));
    CK(cudaMalloc(&d, 256ull << 20));
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, j;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
    std::mt19937_64 rng(1);
    std::vector<void*> dst(nb), src(nb);
    std::vector<size_t> sz(nb, blk);
    for (int mode = 0; mode < 4; ++mode) {
        float best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(e0, s0));
            for (size_t st = 0; st < steps; ++st) {
                for (size_t i = 0; i < nb; ++i) {
                    src[i] = static_cast<char*>(h) + (rng() % (img / blk - 1)) * blk + (rng() % 4096) * 16;
                    dst[i] = static_cast<char*>(d) + ((st % 3) * nb + i) * blk;
                }
                if (mode == 0) {
                    for (size_t i = 0; i < nb; ++i) CK(cudaMemcpyAsync(dst[i], src[i], blk, cudaMemcpyHostToDevice, s0));
                } else if (mode == 1 || mode == 2) {
                    cudaMemcpyAttributes attr{};
                    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
                    attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
                    size_t ai = 0, fi = 0;
                    const size_t h1 = mode == 2 ? nb / 2 : nb;
                    CK(cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), h1, &attr, &ai, 1, &fi, s0));
                    if (mode == 2) {
                        CK(cudaMemcpyBatchAsync(dst.data() + h1, src.data() + h1, sz.data() + h1, nb - h1, &attr, &ai, 1,
                                                &fi, s1));
                        CK(cudaEventRecord(j, s1));
                        CK(cudaStreamWaitEvent(s0, j, 0));
                    }
                } else {
                    CK(cudaMemcpyAsync(dst[0], static_cast<char*>(h) + (st % 8) * nb * blk, nb * blk,
                                       cudaMemcpyHostToDevice, s0));
                }
            }
            CK(cudaEventRecord(e1, s0));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const float gbs = steps * nb * blk / (ms / 1e3f) / 1e9f;
            if (gbs > best) best = gbs;
        }
        const char* names[] = {"64 x cudaMemcpyAsync (1 MB)", "cudaMemcpyBatchAsync (64 x 1 MB)",
                               "2 streams x cudaMemcpyBatchAsync (32 x 1 MB)", "one 64 MB cudaMemcpyAsync"};
        std::printf("{\"pattern\": \"%s\", \"GBps\": %.2f}\n", names[mode], best);
    }
    return 0;
}
