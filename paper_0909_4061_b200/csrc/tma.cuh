// TMA descriptor helper shared by the tensor-memory-accelerator kernels
// (gemm_f32_tc.cu, gemm_f64_tma.cu).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace lr {

// 2-D tensor map over a row-major matrix: `inner` elements per row (the
// contiguous dimension), `outer` rows, row stride `row_bytes`; box
// box_inner x box_outer elements.
CUtensorMap make_map_2d(CUtensorMapDataType dt, const void* ptr, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                        CUtensorMapSwizzle swz);

}  // namespace lr
