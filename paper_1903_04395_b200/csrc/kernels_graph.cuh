// kernels_graph.cuh -- per-graph preparation on the device (tcg_set_graph):
// the whole-row SpMM segment schedule and the degree order of the row
// bucketing, built from the uploaded row_ptr so a new CSR costs its H2D copy
// plus a few O(n) kernels (no host pass over the rows, no per-call
// cudaMalloc).  Same schedules as the host builder (build_schedule): rows cut
// into segments of <= kSegMax neighbours, stably sorted by length
// (descending); rows longer than kSegMax get fp64 partial slots numbered in
// row order; hub rows (> kBucketLong) cut into kLongChunk chunks in degree
// order.
#pragma once

namespace tcg {
namespace dev {

// per row: segment count, partial-slot count, split flag, degree-order key
__global__ void graph_row_counts(const int64_t* __restrict__ row_ptr, int32_t n, int32_t* __restrict__ nseg,
                                 int32_t* __restrict__ nslot, int32_t* __restrict__ split,
                                 uint32_t* __restrict__ okey, int32_t* __restrict__ ids, int32_t* __restrict__ nsmall) {
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v > n) return;
  if (v == n) {  // the scans' last element: totals
    nseg[n] = nslot[n] = split[n] = 0;
    return;
  }
  const int64_t d = row_ptr[v + 1] - row_ptr[v];
  const int32_t s = d <= kSegMax ? 1 : static_cast<int32_t>((d + kSegMax - 1) / kSegMax);
  nseg[v] = s;
  nslot[v] = d > kSegMax ? s : 0;
  split[v] = d > kSegMax ? 1 : 0;
  okey[v] = ~static_cast<uint32_t>(d);  // ascending key = descending degree (stable: ascending id)
  ids[v] = static_cast<int32_t>(v);
  const unsigned big = __ballot_sync(__activemask(), d > kBucketSmall);
  if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && big) atomicAdd(nsmall, __popc(big));
}

// segments of row v at seg_off[v]: key = kSegMax - len (ascending = longest first)
__global__ void graph_emit_segs(const int64_t* __restrict__ row_ptr, int32_t n, const int32_t* __restrict__ seg_off,
                                const int32_t* __restrict__ slot_off, const int32_t* __restrict__ split_off,
                                Seg* __restrict__ segs, uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                int32_t* __restrict__ split_rows, int32_t* __restrict__ slot_begin,
                                int32_t* __restrict__ slot_row) {
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t b = row_ptr[v], d = row_ptr[v + 1] - b;
  const int32_t o = seg_off[v];
  if (d <= kSegMax) {
    segs[o] = Seg{b, static_cast<int32_t>(d), static_cast<int32_t>(v)};
    keys[o] = static_cast<uint32_t>(kSegMax - d);
    vals[o] = o;
    return;
  }
  const int32_t so = slot_off[v], r = split_off[v];
  split_rows[r] = static_cast<int32_t>(v);
  slot_begin[r] = so;
  for (int64_t q = 0, j = 0; q < d; q += kSegMax, ++j) {
    const int32_t len = static_cast<int32_t>(min(static_cast<int64_t>(kSegMax), d - q));
    segs[o + j] = Seg{b + q, len, -1 - (so + static_cast<int32_t>(j))};
    keys[o + j] = static_cast<uint32_t>(kSegMax - len);
    vals[o + j] = o + static_cast<int32_t>(j);
    slot_row[so + j] = static_cast<int32_t>(v);
  }
}

// sorted schedule, padded with no-op segments to nseg_padded
__global__ void graph_gather_segs(const Seg* __restrict__ segs, const int32_t* __restrict__ perm, int64_t nseg,
                                  int64_t nseg_padded, Seg* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nseg_padded) return;
  out[i] = i < nseg ? segs[perm[i]] : Seg{0, 0, kSkip};
}

// hub rows (the first nlong of the degree order): chunk counts, then chunks
__global__ void graph_long_counts(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ order, int32_t nlong,
                                  int32_t* __restrict__ nch) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > nlong) return;
  if (r == nlong) { nch[r] = 0; return; }
  const int32_t v = order[r];
  const int64_t d = row_ptr[v + 1] - row_ptr[v];
  nch[r] = static_cast<int32_t>((d + kLongChunk - 1) / kLongChunk);
}
__global__ void graph_long_chunks(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ order, int32_t nlong,
                                  const int32_t* __restrict__ first, int4* __restrict__ chunks) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nlong) return;
  const int32_t v = order[r];
  const int64_t d = row_ptr[v + 1] - row_ptr[v];
  int32_t q = 0;
  for (int64_t o = 0; o < d; o += kLongChunk, ++q)
    chunks[first[r] + q] = make_int4(v, static_cast<int32_t>(o), static_cast<int32_t>(min(d, o + kLongChunk)), q);
}

// ------------------------------------------------------- CSR from edges
// graph.hpp:65-95 from_edges on the device: every (u, v) edge becomes the two
// directed keys u << b | v and v << b | u (b = bits of n); one radix sort, then
// a key survives if it differs from its predecessor (dedup) and is not a
// self-loop; its high part counts toward row u, its low part is the column.
// Rows come out ascending, symmetric, loop- and duplicate-free -- the
// reference's CSR.  ids out of range are flagged (bad = 1).
__global__ void edges_minmax(const int32_t* __restrict__ e, int64_t cnt, int32_t* __restrict__ mx,
                             int32_t* __restrict__ mn) {
  int32_t a = INT32_MIN, b = INT32_MAX;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    a = max(a, e[i]);
    b = min(b, e[i]);
  }
  for (int o = 16; o; o >>= 1) {
    a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = min(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(mx, a);
    atomicMin(mn, b);
  }
}
__global__ void edges_keys(const int32_t* __restrict__ e, int64_t m, int bits, uint64_t* __restrict__ keys) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t u = static_cast<uint32_t>(e[2 * i]), v = static_cast<uint32_t>(e[2 * i + 1]);
    keys[2 * i] = u << bits | v;
    keys[2 * i + 1] = v << bits | u;
  }
}
// keep[i] = first of its run and not a self-loop; deg[u] += keep
__global__ void edges_keep(const uint64_t* __restrict__ k, int64_t cnt, int bits, int32_t* __restrict__ keep,
                           int64_t* __restrict__ deg) {
  const uint64_t lo = (uint64_t{1} << bits) - 1;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t x = k[i];
    const uint64_t u = x >> bits, v = x & lo;
    const bool ok = u != v && (i == 0 || k[i - 1] != x);
    keep[i] = ok;
    if (ok) atomicAdd(reinterpret_cast<unsigned long long*>(deg + u), 1ull);
  }
}
__global__ void edges_emit(const uint64_t* __restrict__ k, const int32_t* __restrict__ keep,
                           const int32_t* __restrict__ pos, int64_t cnt, int bits, int32_t* __restrict__ col) {
  const uint64_t lo = (uint64_t{1} << bits) - 1;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (keep[i]) col[pos[i]] = static_cast<int32_t>(k[i] & lo);
}

// ---------------------------------------------------------------- relabeling
// Degree-aware relabeling with isolated-vertex compaction (the
// reference's permutation hook is Graph::apply_permutation, graph.hpp:189-207):
// new id = rank in descending degree (stable: ascending old id), isolated
// vertices (degree 0, necessarily last) dropped.  Every count table then has
// n_act rows, and the hub rows every SpMM gathers most often sit in one
// contiguous, L2-resident prefix of each panel.

// key = ~deg (ascending key = descending degree), ids = old id, nact += deg > 0
__global__ void relabel_keys(const int64_t* __restrict__ row_ptr, int32_t n, uint32_t* __restrict__ key,
                             int32_t* __restrict__ ids, int32_t* __restrict__ nact) {
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = v < n && row_ptr[v + 1] > row_ptr[v];
  if (v < n) {
    key[v] = ~static_cast<uint32_t>(row_ptr[v + 1] - row_ptr[v]);
    ids[v] = static_cast<int32_t>(v);
  }
  const unsigned m = __ballot_sync(0xffffffffu, live);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(nact, __popc(m));
}

// inv[perm[i]] = i and deg'[i] = deg(perm[i]) for the nact live rows; deg'[nact] = 0
__global__ void relabel_inverse(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ perm, int32_t nact,
                                int32_t* __restrict__ inv, int64_t* __restrict__ deg) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i > nact) return;
  if (i == nact) { deg[i] = 0; return; }
  const int32_t v = perm[i];
  inv[v] = static_cast<int32_t>(i);
  deg[i] = row_ptr[v + 1] - row_ptr[v];
}

// warp per new row i: col'[rp'[i] + j] = inv[col[rp[perm[i]] + j]] (the
// neighbours of a live vertex are live: the CSR is symmetric)
__global__ void __launch_bounds__(256)
relabel_fill(const int64_t* __restrict__ rp_old, const int32_t* __restrict__ col_old, const int32_t* __restrict__ perm,
             const int32_t* __restrict__ inv, const int64_t* __restrict__ rp_new, int32_t nact, int32_t* __restrict__ col_new) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < nact; i += nw) {
    const int32_t v = perm[i];
    const int64_t b = rp_old[v], d = rp_old[v + 1] - b, o = rp_new[i];
    for (int64_t j = lane; j < d; j += 32) col_new[o + j] = __ldg(inv + __ldg(col_old + b + j));
  }
}

// per coloring: colors of the internal rows, out[i] = in[perm[i]]
__global__ void permute_colors(const uint8_t* __restrict__ in, const int32_t* __restrict__ perm, int32_t n,
                               uint8_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[perm[i]];
}

// per-vertex fp64 results back to the caller's ids: out[perm[i]] = in[i]
// (out pre-zeroed: isolated vertices count 0)
__global__ void scatter_rows_f64(const double* __restrict__ in, const int32_t* __restrict__ perm, int32_t n,
                                 double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[perm[i]] = in[i];
}

}  // namespace dev
}  // namespace tcg
