// Probe: does synccheck report "Missing init" for an mbarrier wait in a warp that also
// ran tcgen05.alloc (the attention kernel's Q-producer pattern)? Same init / fence /
// __syncthreads / parity-1 wait as attention.cu:172-245, plus the TMEM alloc of warp 10.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
struct Bars { uint64_t full[2][2]; uint64_t empty[2][2]; uint32_t tmem; };
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__global__ void __launch_bounds__(384, 1) k(int* out, int use_tmem) {
    extern __shared__ __align__(1024) unsigned char sm[];
    Bars* bar = reinterpret_cast<Bars*>(sm + 200 * 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 8 && lane == 0) {
        for (int s = 0; s < 2; ++s)
            for (int q = 0; q < 2; ++q) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar->full[s][q])), "r"(1));
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar->empty[s][q])), "r"(1));
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (use_tmem && warp == 10) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&bar->tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 10 || warp == 11) {
        const int s = warp - 10;
        if (elect_one()) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(su32(&bar->empty[s][0])), "r"(1u) : "memory");
            out[blockIdx.x * 2 + s] = 1;
        }
    }
    __syncthreads();
    if (use_tmem && warp == 10) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(bar->tmem) : "memory");
    }
}
int main() {
    int* d; cudaMalloc(&d, 64 * sizeof(int));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    k<<<8, 384, 210 * 1024>>>(d, 0);
    cudaError_t e0 = cudaDeviceSynchronize();
    k<<<8, 384, 210 * 1024>>>(d, 1);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mbar+tmem probe: %s / %s\n", cudaGetErrorString(e0), cudaGetErrorString(e));
    return e != cudaSuccess;
}
