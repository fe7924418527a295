// PCIe H2D calibration for the loader's staging pattern: per step, 64 copies of
// ~1 MB blocks from random offsets of a pinned host image (cfg1: f = 64 rows of
// ~16 KB), as 64 cudaMemcpyAsync dealt round-robin over 1 / 2 / 3 / 4 copy
// streams (the loader's copy lanes), against one contiguous copy of the same
// bytes; block sizes 1 MB and 512 KB (cfg1's coded records).
// Build: nvcc -O2 -o h2d_pattern h2d_pattern.cu ; run on the B200 box.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
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
    std::vector<cudaStream_t> lanes(4);
    std::vector<cudaEvent_t> lev(4);
    for (int l = 0; l < 4; ++l) {
        CK(cudaStreamCreateWithFlags(&lanes[l], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&lev[l], cudaEventDisableTiming));
    }
    lanes[0] = s0;
    (void)s1;
    for (size_t bsz : {blk, blk / 2}) {
        for (int mode = 1; mode <= 5; ++mode) {  // 1..4 lanes, 5 = contiguous
            float best = 0;
            for (int rep = 0; rep < 3; ++rep) {
                CK(cudaEventRecord(e0, s0));
                for (size_t st = 0; st < steps; ++st) {
                    if (mode == 5) {
                        CK(cudaMemcpyAsync(d, static_cast<char*>(h) + (st % 8) * nb * bsz, nb * bsz,
                                           cudaMemcpyHostToDevice, s0));
                        continue;
                    }
                    CK(cudaEventRecord(j, s0));
                    for (int l = 1; l < mode; ++l) CK(cudaStreamWaitEvent(lanes[l], j, 0));
                    for (size_t i = 0; i < nb; ++i) {
                        char* src = static_cast<char*>(h) + (rng() % (img / bsz - 1)) * bsz + (rng() % 4096) * 16;
                        char* dst = static_cast<char*>(d) + ((st % 3) * nb + i) * bsz;
                        CK(cudaMemcpyAsync(dst, src, bsz, cudaMemcpyHostToDevice, lanes[i % mode]));
                    }
                    for (int l = 1; l < mode; ++l) {
                        CK(cudaEventRecord(lev[l], lanes[l]));
                        CK(cudaStreamWaitEvent(s0, lev[l], 0));
                    }
                }
                CK(cudaEventRecord(e1, s0));
                CK(cudaEventSynchronize(e1));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                const float gbs = steps * nb * bsz / (ms / 1e3f) / 1e9f;
                if (gbs > best) best = gbs;
            }
            std::printf("{\"pattern\": \"%s\", \"lanes\": %d, \"block_kb\": %zu, \"GBps\": %.2f}\n",
                        mode == 5 ? "one contiguous cudaMemcpyAsync" : "64 x cudaMemcpyAsync round-robin", mode == 5 ? 0 : mode,
                        bsz >> 10, best);
        }
    }
    // host gather: T threads memcpy the step's 64 random blocks into one of two pinned
    // bounce buffers (contiguous), then ONE cudaMemcpyAsync per step; the gather of
    // step s+1 overlaps the DMA of step s
    void* bounce[2];
    CK(cudaHostAlloc(&bounce[0], 64ull << 20, cudaHostAllocDefault));
    CK(cudaHostAlloc(&bounce[1], 64ull << 20, cudaHostAllocDefault));
    cudaEvent_t bev[2];
    CK(cudaEventCreateWithFlags(&bev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&bev[1], cudaEventDisableTiming));
    for (size_t bsz : {blk, blk / 2}) {
        for (unsigned T : {1u, 2u, 4u, 8u, 12u}) {
            float best = 0;
            for (int rep = 0; rep < 3; ++rep) {
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(bev[0], s0));
                CK(cudaEventRecord(bev[1], s0));
                CK(cudaEventRecord(e0, s0));
                for (size_t st = 0; st < steps; ++st) {
                    std::vector<char*> srcs(nb);
                    for (size_t i = 0; i < nb; ++i)
                        srcs[i] = static_cast<char*>(h) + (rng() % (img / bsz - 1)) * bsz + (rng() % 4096) * 16;
                    char* bb = static_cast<char*>(bounce[st & 1]);
                    CK(cudaEventSynchronize(bev[st & 1]));
                    std::vector<std::thread> pool;
                    for (unsigned t = 0; t < T; ++t)
                        pool.emplace_back([&, t] {
                            for (size_t i = t; i < nb; i += T) std::memcpy(bb + i * bsz, srcs[i], bsz);
                        });
                    for (auto& th : pool) th.join();
                    CK(cudaMemcpyAsync(static_cast<char*>(d) + (st % 3) * nb * bsz, bb, nb * bsz,
                                       cudaMemcpyHostToDevice, s0));
                    CK(cudaEventRecord(bev[st & 1], s0));
                }
                CK(cudaEventRecord(e1, s0));
                CK(cudaEventSynchronize(e1));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                const float gbs = steps * nb * bsz / (ms / 1e3f) / 1e9f;
                if (gbs > best) best = gbs;
            }
            std::printf("{\"pattern\": \"host gather (%u threads) + one cudaMemcpyAsync per step\", \"block_kb\": %zu, "
                        "\"GBps\": %.2f}\n", T, bsz >> 10, best);
        }
    }
    return 0;
}
