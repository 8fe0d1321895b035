// Shared helpers for the rsb200 kernels: status/error plumbing, order-preserving key
// transforms, warp reductions. sm_100a only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include "../../include/rsb200.h"
#include <nvtx3/nvToolsExt.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "rsb200 targets sm_100a only"
#endif

namespace rs {

// NVTX range over a C-ABI entry point (nvtx3 is header-only: a no-op unless a profiler
// injects itself), so nsys / ncu --nvtx timelines show the reference-facing calls.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define RS_NVTX() ::rs::NvtxRange rs_nvtx_range_(__func__)


// Thread-local last-error message (set by every failing entry point).
void set_error(const char* fmt, ...);

#define RS_CHECK_ARG(cond, ...)            \
    do {                                   \
        if (!(cond)) {                     \
            ::rs::set_error(__VA_ARGS__);  \
            return RS_ERR_INVALID;         \
        }                                  \
    } while (0)

#define RS_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess) {                                                           \
            ::rs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
            return RS_ERR_CUDA;                                                            \
        }                                                                                  \
    } while (0)

// Every kernel launch is followed by RS_LAUNCH_CHECK(), which also counts it
// (rs_launch_count(): the bench's gpu_launches evidence).
void note_launch();
#define RS_LAUNCH_CHECK()      \
    do {                       \
        ::rs::note_launch();   \
        RS_CUDA(cudaGetLastError()); \
    } while (0)

#define RS_TRY(expr)             \
    do {                         \
        int _s = (expr);         \
        if (_s != RS_OK) return _s; \
    } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device), thread-safe.
cudaError_t ensure_smem(const void* func, int bytes);

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Arena {
    char* base;
    size_t cap;
    size_t used;
    __host__ Arena(void* p, size_t c) : base(static_cast<char*>(p)), cap(c), used(0) {}
    template <typename T>
    __host__ T* take(size_t count) {
        size_t off = align_up(used, 256);
        used = off + count * sizeof(T);
        return reinterpret_cast<T*>(base + off);
    }
    __host__ bool ok() const { return used <= cap; }
};
// Size-only twin of Arena, for *_workspace_size().
struct ArenaSizer {
    size_t used = 0;
    template <typename T>
    void take(size_t count) { used = align_up(used, 256) + count * sizeof(T); }
};

// --- order-preserving integer images of numeric keys ------------------------------
// Comparing the images as unsigned integers gives the same order (and the same ties)
// as comparing the values as float64, which is what the reference does after
// np.asarray(..., dtype=np.float64). -0.0 is canonicalised to +0.0 (they compare
// equal in Python/numpy).
__device__ __forceinline__ uint64_t orderable_f64(double v) {
    if (v == 0.0) v = 0.0;  // -0.0 -> +0.0
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ uint32_t orderable_f32(float v) {
    if (v == 0.0f) v = 0.0f;
    uint32_t b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint32_t orderable_i32(int32_t v) {
    return static_cast<uint32_t>(v) ^ 0x80000000u;
}
__device__ __forceinline__ uint64_t orderable_i64(int64_t v) {
    return static_cast<uint64_t>(v) ^ 0x8000000000000000ull;
}

// SM count of the current device (cached per device ordinal).
inline int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cache[dev] && cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 148;
    return cache[dev];
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace rs
