// layout.hpp -- device data-layout constants shared by host and kernels.
//
// Count tables are fp32 PANELS: a table with C color-set columns is
// P = ceil(C/32) panels of n vertex rows.  Every panel but the last is 32
// floats (128 B = one L2 line) wide; the last is the narrowest of {8,16,32}
// that holds the remaining columns.  Panel p starts at p * n * 32 floats.
#pragma once

#include <cstdint>

namespace tcg {
namespace dev {

constexpr int kZ = 32;           // full panel width (floats)
constexpr int kSegMax = 1024;    // longest neighbour segment one lane group owns
constexpr int kSegPad = 16;      // schedules padded to this many segments
constexpr int kTileV = 32;       // vertices per eMA tile (lane = vertex)

__host__ __device__ inline int last_panel_width(int64_t C) {
  const int r = static_cast<int>(C % kZ);
  return r == 0 ? kZ : (r <= 8 ? 8 : (r <= 16 ? 16 : kZ));
}
__host__ __device__ inline int num_panels(int64_t C) { return static_cast<int>((C + kZ - 1) / kZ); }
__host__ __device__ inline int panel_width(int64_t C, int p) {
  return p == num_panels(C) - 1 ? last_panel_width(C) : kZ;
}
// floats from the table base to element (v, c)
__host__ __device__ inline int64_t panel_offset(int64_t C, int64_t n, int64_t v, int64_t c) {
  const int p = static_cast<int>(c / kZ);
  return static_cast<int64_t>(p) * n * kZ + v * panel_width(C, p) + (c % kZ);
}
__host__ __device__ inline int64_t table_floats(int64_t C, int64_t n) {
  return C <= 0 ? 0 : (static_cast<int64_t>(num_panels(C) - 1) * kZ + last_panel_width(C)) * n;
}

struct Seg {                     // one SpMM work unit: part of one adjacency row
  int64_t e_begin;               // first CSR slot
  int32_t len;                   // <= kSegMax neighbours
  int32_t dst;                   // see encoding below
};
// dst encoding: row r (0 <= r < n) written directly; dst == kSkip: padding;
// dst <= -1: fp64 partial slot (-1 - dst), summed by spmm_fixup.
constexpr int32_t kSkip = 0x7FFFFFFF;

}  // namespace dev
}  // namespace tcg
