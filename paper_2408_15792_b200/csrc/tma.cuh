// Host-side TMA tensor-map encoding (driver entry point resolved at rs_device_init).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"

namespace rs {
extern PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled;
int resolve_tma_encoder();

// 2-D bf16 map over a row-major [rows, cols] matrix with the given row pitch; box
// [box_rows, box_cols] (box_cols * 2 bytes must equal the swizzle span for SW128).
static inline int make_tmap_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                                 uint64_t row_pitch_bytes, uint32_t box_rows, uint32_t box_cols,
                                 CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    if (!g_encode_tiled) {
        int s = resolve_tma_encoder();
        if (s != RS_OK) return s;
    }
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {row_pitch_bytes};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d): rows=%llu cols=%llu pitch=%llu box=%ux%u", (int)r,
                  (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)row_pitch_bytes,
                  box_rows, box_cols);
        return RS_ERR_INVALID;
    }
    return RS_OK;
}
// Generic 2-D map (any element type) for TMA stores of epilogue sub-tiles.
static inline int make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, uint32_t esize, uint64_t rows,
                               uint64_t cols, uint64_t row_pitch_bytes, uint32_t box_rows, uint32_t box_cols,
                               CUtensorMapSwizzle sw) {
    if (!g_encode_tiled) {
        int s = resolve_tma_encoder();
        if (s != RS_OK) return s;
    }
    (void)esize;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {row_pitch_bytes};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode_tiled(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (store) failed (%d)", (int)r);
        return RS_ERR_INVALID;
    }
    return RS_OK;
}
}  // namespace rs
