// tma.cuh -- host-side TMA tensor-map encoding (driver entry point fetched at
// run time through cudart, so the library does not link libcuda).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace hf {

// 2-D fp32 row table [rows][cols] (row stride cols*4 B) for gather4: box
// {box_cols, 1}, 128-byte swizzle.
bool tma_map_rows(CUtensorMap* map, const float* base, long long rows, int cols, int box_cols);
// 3-D fp32 [n][rows][cols] for tile loads: box {box_cols, box_rows, 1}, 128-byte swizzle.
bool tma_map_3d(CUtensorMap* map, const float* base, int n, int rows, int cols, int box_cols,
                int box_rows);

}  // namespace hf
