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

// rank-D tensor map (rank <= 5): dims[0] contiguous, byte strides of dims
// 1..rank-1, box sizes.
CUtensorMap make_map_nd(CUtensorMapDataType dt, const void* ptr, int rank, const uint64_t* dims,
                        const uint64_t* strides, const uint32_t* box, CUtensorMapSwizzle swz);
// 3-D tensor map: dims[0] contiguous, byte strides of dims 1 and 2, box sizes.
CUtensorMap make_map_3d(CUtensorMapDataType dt, const void* ptr, const uint64_t dims[3],
                        const uint64_t strides[2], const uint32_t box[3], CUtensorMapSwizzle swz);

}  // namespace lr
