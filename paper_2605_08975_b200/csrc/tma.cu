// TMA tensor-map construction (driver entry point resolved at run time so the
// library links only against cudart).
#include <cudaTypedefs.h>

#include "ctx.h"

namespace alpa {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        ALPA_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess)
            fail(ALPA_ERR_INTERNAL, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D bf16 row-major tensor [outer][inner] (row stride in bytes), box
// {box_inner, box_outer}, SWIZZLE_128B (box_inner * 2 must be 128).
void make_tmap_bf16_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                       uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(ALPA_ERR_INTERNAL, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// 2-D fp32 row-major tensor [outer][inner], box {box_inner (<= 256), box_outer},
// no swizzle (epilogue TMA stores of fp32 rows staged row-major in smem).
void make_tmap_f32_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(ALPA_ERR_INTERNAL, "cuTensorMapEncodeTiled (f32) failed (" + std::to_string((int)r) + ")");
}

// 3-D fp32 tensor [d2][d1][d0] (strides in bytes), box {32, box1, 1}, SWIZZLE_128B:
// the attention KV-split partials [split][token][kv], one 128-byte swizzled
// panel of 32 fp32 per box row; the split dimension keeps out-of-range token
// rows of one split from landing in the next split's rows (TMA clips per dim).
void make_tmap_f32_3d_sw128(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                            uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box1) {
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
    cuuint32_t box[3] = {32, box1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(ALPA_ERR_INTERNAL, "cuTensorMapEncodeTiled (f32 3d) failed (" + std::to_string((int)r) + ")");
}

// 3-D "panel" view of a row-major [rows][cols] tensor for one-instruction stores of
// a 16-row chunk across several 128-byte panels: dims {panel elems, rows, cols /
// panel elems}, strides {row bytes, 128 B}, box {panel elems, box_rows, panels},
// SWIZZLE_128B.  The smem box is [panels][box_rows][128 B] (chunk-major staging).
void make_tmap_panels(CUtensorMap* m, const void* base, bool f32, uint64_t cols, uint64_t rows,
                      uint64_t row_stride_bytes, uint32_t box_rows, uint32_t panels) {
    const uint64_t pe = f32 ? 32 : 64;  // elements per 128-byte panel row
    cuuint64_t dims[3] = {pe, rows, cols / pe};
    cuuint64_t strides[2] = {row_stride_bytes, 128};
    cuuint32_t box[3] = {(cuuint32_t)pe, box_rows, panels};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(ALPA_ERR_INTERNAL, "cuTensorMapEncodeTiled (panels) failed (" + std::to_string((int)r) + ")");
}

}  // namespace alpa
