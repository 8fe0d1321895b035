// Error state, versioning and device init for librsb200.
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <atomic>
#include <map>
#include <mutex>
#include <utility>
#include "common.cuh"
#include "tma.cuh"

namespace rs {
static thread_local char g_err[1024] = {0};
void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Dynamic shared-memory opt-in, tracked per (kernel, device): the attribute is per
// device, so a process driving several GPUs sets it once on each.
cudaError_t ensure_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    int& have = done[{func, dev}];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

int resolve_tma_encoder() {
    if (g_encode_tiled) return RS_OK;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    RS_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000,
                                             cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || fn == nullptr) {
        set_error("cuTensorMapEncodeTiled entry point not found");
        return RS_ERR_UNSUPPORTED;
    }
    g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return RS_OK;
}
}  // namespace rs

extern "C" const char* rs_last_error(void) { return rs::g_err; }
extern "C" int rs_version(void) { return 1; }
extern "C" uint64_t rs_launch_count(void) { return rs::g_launches.load(); }

extern "C" int rs_device_init(int device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
    RS_NVTX();
    RS_CUDA(cudaSetDevice(device));
    cudaDeviceProp p;
    RS_CUDA(cudaGetDeviceProperties(&p, device));
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    if (p.major != 10) {
        rs::set_error("rsb200 is built for sm_100a; device %d is sm_%d%d", device, p.major, p.minor);
        return RS_ERR_UNSUPPORTED;
    }
    return rs::resolve_tma_encoder();
}
