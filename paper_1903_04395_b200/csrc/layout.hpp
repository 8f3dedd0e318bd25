// layout.hpp -- device data-layout constants shared by host and kernels.
#pragma once

#include <cstdint>

namespace tcg {
namespace dev {

constexpr int Z = 16;            // panel width (floats)
constexpr int kSegMax = 1024;    // longest neighbour segment one 4-lane group owns
constexpr int kTileV = 32;       // vertices per eMA tile (lane = vertex)
constexpr int kEmaWarps = 8;

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
