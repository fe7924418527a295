// Probe: how large a page-locked host region this box allows, by method.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
int main(int argc, char** argv) {
    for (int i = 1; i < argc; ++i) {
        const size_t gb = strtoull(argv[i], nullptr, 10);
        const size_t n = gb << 30;
        auto t0 = std::chrono::steady_clock::now();
        void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
        memset(p, 1, n);
        auto t1 = std::chrono::steady_clock::now();
        cudaError_t rc = cudaHostRegister(p, n, cudaHostRegisterPortable);
        auto t2 = std::chrono::steady_clock::now();
        printf("mmap+touch %zu GB %.1fs register rc=%d (%s) %.1fs\n", gb, std::chrono::duration<double>(t1 - t0).count(),
               rc, cudaGetErrorString(rc), std::chrono::duration<double>(t2 - t1).count());
        cudaGetLastError();
        if (rc == cudaSuccess) cudaHostUnregister(p);
        munmap(p, n);
        // same with MAP_POPULATE-less shared anonymous
        void* h = nullptr;
        t1 = std::chrono::steady_clock::now();
        rc = cudaHostAlloc(&h, n, cudaHostAllocPortable);
        t2 = std::chrono::steady_clock::now();
        printf("cudaHostAlloc %zu GB rc=%d (%s) %.1fs\n", gb, rc, cudaGetErrorString(rc),
               std::chrono::duration<double>(t2 - t1).count());
        cudaGetLastError();
        if (rc == cudaSuccess) cudaFreeHost(h);
        fflush(stdout);
    }
}
