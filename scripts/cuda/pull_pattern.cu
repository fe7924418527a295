// Host -> HBM staging by the SMs instead of the copy engine: per step, 64 blocks
// of 512 KB / 1 MB from random 16-B aligned offsets of a 1.6 GB mapped pinned
// image (the cfg1 loader's staging pattern) gathered into HBM by
//   ld  : a kernel of plain 16-B loads (U loads in flight per thread), or
//   tma : 1-D TMA bulk loads host -> shared (S stages of P bytes per CTA, mbarrier
//         completion) + bulk stores shared -> HBM,
// against one cudaMemcpyAsync per block and one contiguous copy.  Also the copy
// engine and the TMA pull side by side (half the blocks each, two streams).
// Build: nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o pull_pattern pull_pattern.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Job {
    const uint8_t* src;
    uint8_t* dst;
    uint64_t bytes;
};
constexpr int kMaxJobs = 64;
struct Jobs {
    int n;
    Job j[kMaxJobs];
};

template <int U>
__global__ void __launch_bounds__(256) k_pull_ld(const __grid_constant__ Jobs jobs) {
    // blockIdx.y = job; blockIdx.x strides over the job's 16-B chunks
    const Job jb = jobs.j[blockIdx.y];
    const uint64_t n = jb.bytes / 16;
    const uint4* s = reinterpret_cast<const uint4*>(jb.src);
    uint4* d = reinterpret_cast<uint4*>(jb.dst);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 256;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += stride * U) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i + k * stride < n)
                asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                             : "l"(s + i + k * stride));
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i + k * stride < n) d[i + k * stride] = v[k];
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// one elected thread per CTA streams the CTA's share of the job in P-byte pieces
// through S shared stages
__global__ void __launch_bounds__(32) k_pull_tma(const __grid_constant__ Jobs jobs, uint32_t P, uint32_t S) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[16];
    if (threadIdx.x != 0) return;
    const Job jb = jobs.j[blockIdx.y];
    const uint64_t pieces = (jb.bytes + P - 1) / P;
    for (uint32_t s = 0; s < S; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase[16] = {0};
    // my pieces: blockIdx.x, + gridDim.x, ...
    uint64_t issue = blockIdx.x, done = blockIdx.x;
    uint32_t in_flight = 0, slot_issue = 0, slot_done = 0;
    auto load = [&](uint64_t p, uint32_t slot) {
        const uint32_t bytes = static_cast<uint32_t>((P < jb.bytes - p * P ? (uint64_t)P : jb.bytes - p * P));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[slot])), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(smem + slot * P)),
                     "l"(jb.src + p * P), "r"(bytes), "r"(smem_u32(&bar[slot]))
                     : "memory");
    };
    while (issue < pieces && in_flight < S) {
        load(issue, slot_issue);
        issue += gridDim.x;
        slot_issue = (slot_issue + 1) % S;
        ++in_flight;
    }
    while (done < pieces) {
        // wait for the oldest piece, store it, then reuse its stage once the store has read it
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar[slot_done])), "r"(phase[slot_done])
                         : "memory");
        phase[slot_done] ^= 1;
        const uint32_t bytes = static_cast<uint32_t>((P < jb.bytes - done * P ? (uint64_t)P : jb.bytes - done * P));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(jb.dst + done * P),
                     "r"(smem_u32(smem + slot_done * P)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        done += gridDim.x;
        slot_done = (slot_done + 1) % S;
        --in_flight;
        if (issue < pieces) {
            load(issue, slot_issue);
            issue += gridDim.x;
            slot_issue = (slot_issue + 1) % S;
            ++in_flight;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t img = 1600ull << 20, nb = 64, steps = 40;
    uint8_t* h = nullptr;
    uint8_t* d = nullptr;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h), img, cudaHostAllocMapped | cudaHostAllocPortable));
    for (size_t o = 0; o < img; o += 4096) h[o] = static_cast<uint8_t>(o >> 12);
    uint8_t* hd = nullptr;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd), h, 0));
    CK(cudaMalloc(&d, 256ull << 20));
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, j;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
    CK(cudaFuncSetAttribute(k_pull_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    std::mt19937_64 rng(1);
    struct Mode {
        const char* name;
        int kind;  // 0 ce per block, 1 ld, 2 tma, 3 ce + tma halves, 4 contiguous ce
        unsigned ctas;  // per job (ld / tma)
        uint32_t P, S;
    };
    std::vector<Mode> modes = {{"ce per block", 0, 0, 0, 0},
                               {"ld U=4", 1, 4, 0, 0},
                               {"ld U=4", 1, 8, 0, 0},
                               {"ld U=8", 1, 8, 0, 0},
                               {"tma 32K x4", 2, 2, 32768, 4},
                               {"tma 32K x4", 2, 4, 32768, 4},
                               {"tma 16K x8", 2, 4, 16384, 8},
                               {"tma 64K x3", 2, 2, 65536, 3},
                               {"ce + tma 32K x4 halves", 3, 4, 32768, 4},
                               {"contiguous ce", 4, 0, 0, 0}};
    for (size_t bsz : {size_t(1) << 20, size_t(512) << 10}) {
        for (const Mode& md : modes) {
            float best = 0;
            bool bad = false;
            for (int rep = 0; rep < 3 && !bad; ++rep) {
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(e0, s0));
                for (size_t st = 0; st < steps; ++st) {
                    Jobs jobs{};
                    jobs.n = nb;
                    for (size_t i = 0; i < nb; ++i) {
                        const size_t off = (rng() % (img / bsz - 1)) * bsz + (rng() % 4096) * 16;
                        jobs.j[i] = {hd + off, d + ((st % 3) * nb + i) * bsz, bsz};
                    }
                    if (md.kind == 0) {
                        for (size_t i = 0; i < nb; ++i)
                            CK(cudaMemcpyAsync(jobs.j[i].dst, h + (jobs.j[i].src - hd), bsz, cudaMemcpyHostToDevice, s0));
                    } else if (md.kind == 1) {
                        if (md.name[4] == '8') k_pull_ld<8><<<dim3(md.ctas, nb), 256, 0, s0>>>(jobs);
                        else k_pull_ld<4><<<dim3(md.ctas, nb), 256, 0, s0>>>(jobs);
                    } else if (md.kind == 2) {
                        k_pull_tma<<<dim3(md.ctas, nb), 32, md.P * md.S, s0>>>(jobs, md.P, md.S);
                    } else if (md.kind == 3) {
                        Jobs half = jobs;
                        half.n = nb / 2;
                        for (int i = 0; i < half.n; ++i) half.j[i] = jobs.j[nb / 2 + i];
                        CK(cudaEventRecord(j, s0));
                        CK(cudaStreamWaitEvent(s1, j, 0));
                        k_pull_tma<<<dim3(md.ctas, half.n), 32, md.P * md.S, s1>>>(half, md.P, md.S);
                        for (size_t i = 0; i < nb / 2; ++i)
                            CK(cudaMemcpyAsync(jobs.j[i].dst, h + (jobs.j[i].src - hd), bsz, cudaMemcpyHostToDevice, s0));
                        CK(cudaEventRecord(j, s1));
                        CK(cudaStreamWaitEvent(s0, j, 0));
                    } else {
                        CK(cudaMemcpyAsync(d, h + (st % 8) * nb * bsz, nb * bsz, cudaMemcpyHostToDevice, s0));
                    }
                }
                CK(cudaEventRecord(e1, s0));
                const cudaError_t rc = cudaEventSynchronize(e1);
                if (rc != cudaSuccess) {
                    std::printf("{\"mode\": \"%s\", \"error\": \"%s\"}\n", md.name, cudaGetErrorString(rc));
                    return 1;
                }
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                const float gbs = steps * nb * bsz / (ms / 1e3f) / 1e9f;
                if (gbs > best) best = gbs;
            }
            std::printf("{\"mode\": \"%s\", \"ctas_per_block\": %u, \"block_kb\": %zu, \"GBps\": %.2f}\n", md.name, md.ctas,
                        bsz >> 10, best);
            std::fflush(stdout);
        }
    }
    // correctness of the TMA pull: one step, compare
    {
        Jobs jobs{};
        jobs.n = 8;
        for (int i = 0; i < 8; ++i) jobs.j[i] = {hd + 4096 * 7 * (i + 1) + 48, d + i * (1 << 20), (1u << 20) - 48};
        k_pull_tma<<<dim3(4, 8), 32, 32768 * 4, s0>>>(jobs, 32768, 4);
        CK(cudaStreamSynchronize(s0));
        std::vector<uint8_t> back(1 << 20);
        int bad = 0;
        for (int i = 0; i < 8; ++i) {
            CK(cudaMemcpy(back.data(), d + i * (1 << 20), (1u << 20) - 48, cudaMemcpyDeviceToHost));
            for (size_t k = 0; k < (1u << 20) - 48; ++k) bad += back[k] != h[4096 * 7 * (i + 1) + 48 + k];
        }
        std::printf("{\"tma_pull_check_mismatches\": %d}\n", bad);
    }
    return 0;
}
