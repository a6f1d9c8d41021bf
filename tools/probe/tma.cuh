// TMA tile movement for the sample-major passes: the [E][32-sample] tiles of
// the pitched per-(epoch, sample) rows arrive in shared memory as ONE 2-D bulk tensor copy per
// tile (cp.async.bulk.tensor, completion on an mbarrier), instead of E x 32 per-element
// cp.async / loads.  Rows are pitched to Fp (a multiple of 16 samples, common.cuh pitch16), so
// every row stride is a multiple of 64 B as the tensor map requires.
//
// Shared layout: the box lands row-major [rows][box_cols] with the 128-B (or 64-B) swizzle,
// i.e. the 16-B chunk c of row r sits at chunk c ^ (r & 7) (128-B rows) /
// c ^ ((r >> 1) & 3) (64-B rows).  Readers take 16-B (8-B) chunks with lanes = rows: the
// eight lanes of an LDS.128 phase hit eight distinct chunks, conflict-free.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace clairplan {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// barrier init visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// bounded: a copy that never completes (a bad map) traps the kernel -- a launch error the
// build reports -- instead of hanging the device
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    for (uint32_t n = 0; !mbar_try_wait(bar, parity); ++n)
        if (n == (1u << 22)) __trap();
}

// box at (col, row) of the 2-D map -> dst (1024-B aligned for the 128-B swizzle)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t col, int32_t row,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(smem_u32(bar))
        : "memory");
}

// 16-B chunk q (samples 4q..4q+3) of row e of a 128-B-swizzled [rows][32] u32 tile
__device__ __forceinline__ uint4 tile_quad(const uint32_t* tile, uint32_t e, uint32_t q) {
    return *reinterpret_cast<const uint4*>(tile + e * 32 + ((q ^ (e & 7)) << 2));
}

__device__ __forceinline__ uint32_t quad_at(const uint4& v, int j) {
    return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

// single elements (lanes = rows, one column: 4-way bank conflicts, 8 distinct chunks)
__device__ __forceinline__ uint32_t tile_u32(const uint32_t* tile, uint32_t e, uint32_t s) {
    return tile[e * 32 + ((((s >> 2) ^ (e & 7))) << 2) + (s & 3)];
}
// 64-B-swizzled [rows][32] u16 tile
__device__ __forceinline__ uint16_t tile_u16(const uint16_t* tile, uint32_t e, uint32_t s) {
    return tile[e * 32 + ((((s >> 3) ^ ((e >> 1) & 3))) << 3) + (s & 7)];
}

// 2-D map over rows x cols elements of `elem` bytes, row pitch `pitch_bytes`, box
// box_rows x box_cols, 128-B swizzle when a box row is 128 B, 64-B when it is 64 B.
// Out-of-range elements of a box (cols >= `cols`) arrive as zeros.
inline bool encode_tile_map(CUtensorMap* map, const void* base, uint32_t elem, uint64_t cols, uint64_t rows,
                            uint64_t pitch_bytes, uint32_t box_cols, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    const int promo = 1;  // 128-B rows: no promotion past them
    if (!fn || box_rows == 0 || box_rows > 256 || (pitch_bytes & 15)) return false;
    const CUtensorMapDataType dt = elem == 4   ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                   : elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                               : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    const uint32_t row_bytes = box_cols * elem;
    const CUtensorMapSwizzle sw = row_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                    : CU_TENSOR_MAP_SWIZZLE_NONE;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {pitch_bytes};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
              promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
              : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                           : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace clairplan
