// Host-side TMA tensor maps (qkv_gemm.cu): 2-D bf16 row-major [rows][cols],
// box [box_rows][box_cols], 128-byte swizzle.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace dsa {
CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int box_rows, int box_cols);
}  // namespace dsa
