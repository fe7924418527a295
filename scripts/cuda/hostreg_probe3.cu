// Probe: does a pageable cudaMemcpy from an mmap'd range break a later
// cudaHostRegister of a new mapping at the same address?
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstring>
int main() {
    const size_t n = 2ull << 30;
    void* d = nullptr;
    cudaMalloc(&d, n);
    char* a = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0));
    memset(a, 1, n);
    cudaError_t rc = cudaMemcpy(d, a, n, cudaMemcpyHostToDevice);
    printf("pageable copy rc=%d\n", rc);
    munmap(a, n);
    char* b = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0));
    memset(b, 2, n);
    rc = cudaHostRegister(b, n, cudaHostRegisterPortable);
    printf("same VA %d; register after pageable copy rc=%d (%s)\n", a == b, rc, cudaGetErrorString(rc));
    cudaGetLastError();
    char* c = static_cast<char*>(mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0));
    memset(c, 3, n);
    rc = cudaHostRegister(c, n, cudaHostRegisterPortable);
    printf("fresh VA: register rc=%d (%s)\n", rc, cudaGetErrorString(rc));
    return 0;
}
