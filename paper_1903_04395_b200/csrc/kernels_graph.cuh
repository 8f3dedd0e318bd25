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

}  // namespace dev
}  // namespace tcg
