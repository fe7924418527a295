// Probe: the staging-image pattern -- reserve R GB (MAP_NORESERVE), fill F GB,
// unmap the tail, cudaHostRegister the filled part.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
int main(int argc, char** argv) {
    const size_t R = strtoull(argv[1], nullptr, 10) << 30, F = strtoull(argv[2], nullptr, 10) << 30;
    const int unmap_tail = argc > 3 ? atoi(argv[3]) : 1;
    char* p = static_cast<char*>(mmap(nullptr, R, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0));
    if (p == MAP_FAILED) { printf("mmap failed\n"); return 1; }
    memset(p, 1, F);
    if (unmap_tail) munmap(p + F, R - F);
    auto t0 = std::chrono::steady_clock::now();
    cudaError_t rc = cudaHostRegister(p, F, cudaHostRegisterPortable);
    auto t1 = std::chrono::steady_clock::now();
    printf("reserve %zu GB fill %zu GB unmap_tail %d: register rc=%d (%s) %.1fs\n", R >> 30, F >> 30, unmap_tail, rc,
           cudaGetErrorString(rc), std::chrono::duration<double>(t1 - t0).count());
    return 0;
}
