// Does compute-sanitizer synccheck model mbarrier.init + try_wait.parity? A minimal
// kernel with the same init / fence / __syncthreads / parity-wait pattern as the
// attention and GEMM kernels (one producer thread, one waiter, TMA-free).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int* out, int big) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (big ? 200 * 1024 : 0));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 32) {
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(su32(bar)), "r"(1u) : "memory");
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
        ok = 0;
        while (!ok) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(su32(bar)), "r"(0u) : "memory");
        }
        out[blockIdx.x] = 1;
    }
}
int main() {
    int* d; cudaMalloc(&d, 64 * sizeof(int));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    k<<<8, 64, 1024>>>(d, 0);
    k<<<8, 64, 210 * 1024>>>(d, 1);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mbar probe: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
