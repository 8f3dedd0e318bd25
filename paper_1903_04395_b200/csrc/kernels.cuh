// kernels.cuh -- the sm_100a kernels of one coloring (SURVEY 2.1 kernel inventory).
//
//   mt_coloring  random_coloring (count_table.hpp:90-99): MT19937-64, one CTA
//                per seed, one barrier per 156 words (generation recurrence),
//                rejection handled exactly by a block scan
//   spmm_part    SpMM of the CSR adjacency against one panel of a passive
//                table (la_kernels.hpp:83-102), restricted to one vertex-range
//                PART of the gather source so the gathered rows stay L2
//                resident; lane groups gather 128 B (32-float) rows; fp64
//                accumulation; parts accumulate into the output in order.
//                ONEHOT: the passive child is a leaf (one-hot colors,
//                count_table.hpp:102-107) and the gather reads 1-byte colors
//                -- the neighbour color histogram
//   spmm_fixup   deterministic sum of the fp64 partials of split (hub) rows
//   ema_node     fused eMA color-set combine (engines.hpp:252-268 +
//                la_kernels.hpp:106-114) by parent column; 32-vertex tiles
//                staged in smem, lane = vertex, 8 parent columns per warp in
//                flight; active-leaf variant is a pure gather
//   ema_root     the root node: fp64 per-vertex counts + per-tile fp64 totals
//   root_reduce  deterministic fp64 total (engines.hpp:125-129)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

#include "layout.hpp"

namespace tcg {
namespace dev {

// ------------------------------------------------------------ load helpers
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ld_stream_i32(const int32_t* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// base + idx * bytes as one IMAD.WIDE.U32 (row gathers: idx < 2^27)
__device__ __forceinline__ const float* row_addr(const char* base, uint32_t idx, uint32_t bytes) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(idx), "r"(bytes), "l"(base));
  return reinterpret_cast<const float*>(r);
}
__device__ __forceinline__ float4 ld_keep_f4(const float* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream_f4(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// ------------------------------------------------------------ MT19937-64
// std::mt19937_64 ([rand.predef]) as a word sequence: for j >= 312,
//   x[j] = x[j-156] ^ twist(x[j-312] & UPPER | x[j-311] & LOWER),
// which is libstdc++'s _M_gen_rand unrolled.  Word j of "generation"
// g = j / 156 depends only on generations g-1 and g-2, so 156 threads
// produce 156 words per step with ONE barrier, keeping three generations in
// a shared-memory ring.  Output word o is sequence word 312 + o.  Each word
// is tempered, tested against Rng::below's threshold (rng.hpp:21-27) and
// reduced mod k with a multiply-high (M = floor((2^64-1)/k), one correction).
// Accepted words map to consecutive vertices; a rejection (p <= 17*2^-64 per
// draw, or forced by the test hook) takes an exact block-scan path.
constexpr int kMtThreads = 160;

// Two generations per barrier: thread t also produces word t of generation
// g+1 from its own word t of g and word t+1 of g-1; only word 155 needs a
// word of g it does not own (word 0), which thread 155 recomputes from g-1
// and g-2.  Four ring slots: a round reads one pair, writes the other.
__device__ __forceinline__ uint64_t mt_twist(uint64_t c, uint64_t a, uint64_t b) {
  constexpr uint64_t U = 0xFFFFFFFF80000000ULL, L = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  const uint64_t y = (a & U) | (b & L);
  return c ^ (y >> 1) ^ ((y & 1) ? A : 0);
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  return z ^ (z >> 43);
}

__global__ void __launch_bounds__(kMtThreads)
mt_coloring(const uint64_t* __restrict__ seeds, int32_t n, int k, uint64_t limit, uint64_t magic,
            uint8_t* __restrict__ out, int64_t out_stride) {
  __shared__ uint64_t ring[4][156];
  __shared__ int wcnt[2][kMtThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint8_t* colors = out + blockIdx.x * out_stride;
  if (k == 1) {  // count_table.hpp:97: no draws
    for (int32_t v = t; v < n; v += blockDim.x) colors[v] = 0;
    return;
  }
  if (t == 0) {
    uint64_t s = seeds[blockIdx.x];
    ring[0][0] = s;
    for (int j = 1; j < 312; ++j) {
      s = 6364136223846793005ULL * (s ^ (s >> 62)) + j;
      ring[j / 156][j % 156] = s;
    }
  }
  __syncthreads();
  const bool act = t < 156;
  const uint64_t kk = static_cast<uint64_t>(k);
  auto reduce = [&](uint64_t z) {
    const uint64_t q = __umul64hi(z, magic);
    uint64_t r = z - q * kk;
    if (r >= kk) r -= kk;
    return static_cast<uint8_t>(r);
  };
  int64_t base = 0;
  for (int rd = 0; base < n; ++rd) {
    const uint64_t* P2 = ring[(rd & 1) * 2];      // generation g-2
    const uint64_t* P1 = ring[(rd & 1) * 2 + 1];  // generation g-1
    uint64_t* O0 = ring[((rd + 1) & 1) * 2];      // g
    uint64_t* O1 = ring[((rd + 1) & 1) * 2 + 1];  // g+1
    uint64_t z0 = 0, z1 = 0;
    if (act) {
      const uint64_t w0 = mt_twist(P1[t], P2[t], t < 155 ? P2[t + 1] : P1[0]);
      const uint64_t g0w0 = t < 155 ? 0 : mt_twist(P1[0], P2[0], P2[1]);  // word 0 of g (thread 155)
      const uint64_t w1 = mt_twist(w0, P1[t], t < 155 ? P1[t + 1] : g0w0);
      O0[t] = w0;
      O1[t] = w1;
      z0 = mt_temper(w0);
      z1 = mt_temper(w1);
    }
    const bool rej0 = act && z0 >= limit, rej1 = act && z1 >= limit;
    const uint8_t c0 = reduce(z0), c1 = reduce(z1);
    if (!__syncthreads_or(rej0 || rej1)) {
      if (act) {
        if (base + t < n) colors[base + t] = c0;
        if (base + 156 + t < n) colors[base + 156 + t] = c1;
      }
      base += 312;
    } else {  // exact compaction of the accepted words of both generations, in order
      const unsigned b0 = __ballot_sync(0xffffffffu, rej0), b1 = __ballot_sync(0xffffffffu, rej1);
      if (lane == 0) {
        wcnt[0][warp] = __popc(b0);
        wcnt[1][warp] = __popc(b1);
      }
      __syncthreads();
      int pre0 = __popc(b0 & ((1u << lane) - 1u)), pre1 = __popc(b1 & ((1u << lane) - 1u)), tot0 = 0, tot1 = 0;
      for (int w = 0; w < kMtThreads / 32; ++w) {
        if (w < warp) { pre0 += wcnt[0][w]; pre1 += wcnt[1][w]; }
        tot0 += wcnt[0][w];
        tot1 += wcnt[1][w];
      }
      const int64_t v0 = base + t - pre0;
      const int64_t v1 = base + (156 - tot0) + t - pre1;
      if (act && !rej0 && v0 < n) colors[v0] = c0;
      if (act && !rej1 && v1 < n) colors[v1] = c1;
      base += 312 - tot0 - tot1;
      __syncthreads();
    }
  }
}

// Sharded graphs: colors in padded-global order, pad[r*nmax + j] = color of
// global vertex rows[r] + j (0 for pad rows, which have no neighbours).
__global__ void pad_colors(const uint8_t* __restrict__ colors, const int64_t* __restrict__ rows, int64_t nmax,
                           int64_t nsrc, uint8_t* __restrict__ pad) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nsrc) return;
  const int64_t r = i / nmax, j = i % nmax;
  pad[i] = j < rows[r + 1] - rows[r] ? colors[rows[r] + j] : 0;
}

// ----------------------------------------------------------------- SpMM
// One launch = one (panel, part).  A warp owns 32/G segments, one per lane
// group of G = ZW/4 lanes; each lane carries a float4 of the ZW-wide row.
// Segments are sorted by length (descending) on the host, so group 0 of a
// warp has the longest trip count and all groups run nearly the same.
constexpr int kSpmmWarps = 8;

template <int ZW, bool ONEHOT, int R = 8>   // R: neighbours per round
__global__ void __launch_bounds__(kSpmmWarps * 32)
spmm_part(const Seg* __restrict__ segs, int64_t ntasks, const int32_t* __restrict__ col,
          const float* __restrict__ X, const uint8_t* __restrict__ colors, int color_base,
          float* __restrict__ Y, double* __restrict__ partial, int first) {
  constexpr int G = ZW / 4;          // lanes per group
  constexpr int SPW = 32 / G;        // segments per warp
  const int lane = threadIdx.x & 31, g = lane / G, l = lane % G;
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kSpmmWarps + (threadIdx.x >> 5);
  if (task >= ntasks) return;
  const Seg s = segs[task * SPW + g];
  const int maxlen = __shfl_sync(0xffffffffu, s.len, 0);
  const int32_t* cp = col + s.e_begin;
  const uint64_t pstream = policy_evict_first(), pkeep = policy_evict_last();
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  // the next round's neighbour ids are loaded (from HBM) one round ahead, so
  // the index latency overlaps the current round's L2 gathers
  constexpr int NI = R / G > 0 ? R / G : 1;
  int nxt[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int e = i * G + l;
    nxt[i] = e < s.len ? ld_stream_i32(cp + e, pstream) : -1;
  }
  for (int t = 0; t < maxlen; t += R) {
    int idx[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      idx[i] = nxt[i];
      const int e = t + R + i * G + l;
      nxt[i] = e < s.len ? ld_stream_i32(cp + e, pstream) : -1;
    }
    // R independent unpredicated gathers (missing neighbours read row 0 and
    // are masked after the load), summed in fp32 in a fixed tree (exact for
    // integer partial sums < 2^24) and added to the fp64 accumulators once.
    float4 v[R];
    int uu[R];
#pragma unroll
    for (int j = 0; j < R; ++j) uu[j] = __shfl_sync(0xffffffffu, idx[j / G], g * G + (j % G));
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int u = uu[j] < 0 ? 0 : uu[j];
      if (ONEHOT) {
        const int c = static_cast<int>(__ldg(colors + u)) - color_base - 4 * l;
        v[j] = make_float4(c == 0, c == 1, c == 2, c == 3);
      } else {
        v[j] = ld_keep_f4(X + static_cast<int64_t>(u) * ZW + l * 4, pkeep);
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (uu[j] < 0) v[j] = make_float4(0, 0, 0, 0);
#pragma unroll
    for (int w = R / 2; w; w >>= 1)
#pragma unroll
      for (int j = 0; j < w; ++j) {
        v[j].x += v[j + w].x; v[j].y += v[j + w].y; v[j].z += v[j + w].z; v[j].w += v[j + w].w;
      }
    a0 += v[0].x; a1 += v[0].y; a2 += v[0].z; a3 += v[0].w;
  }
  if (s.dst >= 0) {
    if (s.dst != kSkip) {
      float* yp = Y + static_cast<int64_t>(s.dst) * ZW + l * 4;
      if (!first) {
        const float4 o = ld_stream_f4(yp, pstream);
        a0 += o.x; a1 += o.y; a2 += o.z; a3 += o.w;
      }
      st_stream_f4(yp, make_float4(static_cast<float>(a0), static_cast<float>(a1),
                                   static_cast<float>(a2), static_cast<float>(a3)), pstream);
    }
  } else {
    double* pp = partial + (static_cast<int64_t>(-1 - s.dst) * ZW + l * 4);
    reinterpret_cast<double2*>(pp)[0] = make_double2(a0, a1);
    reinterpret_cast<double2*>(pp)[1] = make_double2(a2, a3);
  }
}

constexpr int kEmaWarps = 16;
constexpr int kSpitch = kTileV + 1;  // smem pitch: lane = vertex, conflict-free
template <int kStageU>
__device__ __forceinline__ void stage_tile(const float* __restrict__ T, int C, int32_t n, int64_t v0,
                                           float* dst);

// ------------------------------------------ rooted-color compressed SpMM
// (host.hpp RootedLayout).  Per coloring, every CSR row is re-ordered by
// (part, neighbour color) and each entry packed as u | color << 27, so the
// SpMM walks a row's neighbours in runs of one color: within a run the
// compressed panel slots mean the same parent columns, so the run is summed
// in registers and scattered into the task's F_g accumulators (smem, fp64)
// once per run.
// packed entry = u << 5 | color (n < 2^27): within a round (one color c) the
// row address X + u * ZW * 4 is (X - c * ZW / 8) + entry * ZW / 8, one
// IMAD.WIDE per entry
constexpr uint32_t kPackSentinel = 0xFFFFFFFFu;  // color 31: never a real color (k <= 20)
constexpr int kColorBits = 5;
constexpr uint32_t kColorMask = (1u << kColorBits) - 1u;
__device__ __forceinline__ uint32_t pack_entry(uint32_t u, uint32_t color) { return u << kColorBits | color; }

// Neighbour colors are sorted in the row's ROTATED order: key(c) = (c - cv - 1)
// mod k for a row of color cv, so the run of the row's own color comes last
// and the part cuts stop before it.  Those neighbours only feed the P'
// columns containing c(v), which no consumer reads (M_a[v, Sa] = 0 unless
// c(v) is in Sa), so the rooted SpMM never walks them.
__device__ __forceinline__ int rot_key(int c, int cv, int k) {
  const int r = c - cv - 1;
  return r < 0 ? r + k : r;
}
__device__ __forceinline__ int unrot_key(int r, int cv, int k) {
  const int c = r + cv + 1;
  return c >= k ? c - k : c;
}

// exclusive scan of cnt[0, nkeys) by one warp, in place
__device__ __forceinline__ void warp_exclusive_scan(int* cnt, int nkeys, int lane) {
  int run = 0;
  for (int i0 = 0; i0 < nkeys; i0 += 32) {
    const int x = i0 + lane < nkeys ? cnt[i0 + lane] : 0;
    int incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (i0 + lane < nkeys) cnt[i0 + lane] = run + incl - x;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
}

// Per coloring: every CSR row stably counting-sorted by neighbour color,
// entries packed as u | color << 27, and the row's PART CUTS recorded: the
// rooted SpMM's parts are contiguous color classes [i*k/P, (i+1)*k/P), so
// part i of row v is [cut[v*(P+1)+i], cut[v*(P+1)+i+1]) -- whole color runs,
// and a part's gather footprint is the rows of its colors (~n/P lines).
// Warp per row over row_order[row0, n) (degree order, static round-robin);
// rows of up to kBucketCache * 32 neighbours are held in registers so both
// passes cost one round of loads.  Longer rows: bucket_long.
constexpr int kBucketCache = 16;
constexpr int kBucketLong = 1024;  // rows above this go to bucket_long (CTA per row)
__global__ void __launch_bounds__(256, 4)  // 64 registers: 4 CTAs per SM (the row loads are latency-bound)
bucket_rows(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
            const uint8_t* __restrict__ colors, const uint8_t* __restrict__ rowc, const int32_t* __restrict__ row_order,
            int32_t row0, int32_t n, int k, int nparts, uint32_t* __restrict__ out, int64_t* __restrict__ cuts,
            float* __restrict__ hist, int hzw) {
  extern __shared__ int bsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* cnt = bsm + warp * k;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t ri = row0 + static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp; ri < n; ri += nwarps) {
    const int32_t v = row_order[ri];
    const int64_t b = row_ptr[v], e = row_ptr[v + 1];
    const int d = static_cast<int>(e - b);
    const int cv = rowc[v];
    for (int i = lane; i < k; i += 32) cnt[i] = 0;
    __syncwarp();
    auto write_cuts = [&]() {
      // the exact neighbour color histogram (the P' of a leaf passive child)
      // is the per-key count: cnt[r+1] - cnt[r] after the scan
      if (hist && lane < hzw) {
        const int r = lane < k ? rot_key(lane, cv, k) : 0;
        const int hi = r + 1 < k ? cnt[r + 1] : d;
        hist[static_cast<int64_t>(v) * hzw + lane] = lane < k ? static_cast<float>(hi - cnt[r]) : 0.f;
      }
      if (lane <= nparts) {  // the last cut stops before the own-color run
        const int cb = lane * k / nparts;
        cuts[static_cast<int64_t>(v) * (nparts + 1) + lane] = b + cnt[cb < k ? cb : k - 1];
      }
      __syncwarp();
    };
    if (d <= kBucketCache * 32) {
      int u[kBucketCache], key[kBucketCache];
#pragma unroll
      for (int q = 0; q < kBucketCache; ++q) u[q] = q * 32 + lane < d ? __ldg(col + b + q * 32 + lane) : -1;
#pragma unroll
      for (int q = 0; q < kBucketCache; ++q) key[q] = u[q] >= 0 ? rot_key(colors[u[q]], cv, k) : -1;
#pragma unroll
      for (int q = 0; q < kBucketCache; ++q) {
        if (q * 32 >= d) break;
        const unsigned same = __match_any_sync(0xffffffffu, key[q]);
        if (key[q] >= 0 && (same & lt) == 0) cnt[key[q]] += __popc(same);
        __syncwarp();
      }
      warp_exclusive_scan(cnt, k, lane);
      write_cuts();
#pragma unroll
      for (int q = 0; q < kBucketCache; ++q) {
        if (q * 32 >= d) break;
        const unsigned same = __match_any_sync(0xffffffffu, key[q]);
        const int slot = key[q] >= 0 ? cnt[key[q]] + __popc(same & lt) : 0;
        __syncwarp();
        if (key[q] >= 0) {
          out[b + slot] = pack_entry(static_cast<uint32_t>(u[q]), static_cast<uint32_t>(unrot_key(key[q], cv, k)));
          if ((same & lt) == 0) cnt[key[q]] += __popc(same);
        }
        __syncwarp();
      }
    } else {
      for (int64_t j = b; j < e; j += 32) {
        const bool ok = j + lane < e;
        const int key = ok ? rot_key(colors[col[j + lane]], cv, k) : -1;
        const unsigned same = __match_any_sync(0xffffffffu, key);
        if (ok && (same & lt) == 0) cnt[key] += __popc(same);
        __syncwarp();
      }
      warp_exclusive_scan(cnt, k, lane);
      write_cuts();
      for (int64_t j = b; j < e; j += 32) {
        const bool ok = j + lane < e;
        const int u = ok ? col[j + lane] : 0;
        const int key = ok ? rot_key(colors[u], cv, k) : -1;
        const unsigned same = __match_any_sync(0xffffffffu, key);
        const int slot = ok ? cnt[key] + __popc(same & lt) : 0;
        __syncwarp();
        if (ok) {
          out[b + slot] = pack_entry(static_cast<uint32_t>(u), static_cast<uint32_t>(unrot_key(key, cv, k)));
          if ((same & lt) == 0) cnt[key] += __popc(same);
        }
        __syncwarp();
      }
    }
  }
}

// Rows of degree <= kBucketSmall (the tail of the degree order, row_order
// [row0, n)): one THREAD per row -- a row's <= 8 entries are sorted by
// (color, position) in registers with a sorting network (unique keys, so the
// result is the stable order), then written with the histogram and the cuts.
// Keeps sparse graphs (cfg2: ~30 neighbours per row, 38% isolated) from
// spending a whole warp on a handful of entries.
constexpr int kBucketSmall = 8;
__global__ void __launch_bounds__(256)
bucket_small(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
             const uint8_t* __restrict__ colors, const uint8_t* __restrict__ rowc, const int32_t* __restrict__ row_order,
             int32_t row0, int32_t n, int k, int nparts, uint32_t* __restrict__ out, int64_t* __restrict__ cuts,
             float* __restrict__ hist, int hzw) {
  const int64_t ri = row0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ri >= n) return;
  const int32_t v = row_order[ri];
  const int cv = rowc[v];
  const int64_t b = row_ptr[v];
  const int d = static_cast<int>(row_ptr[v + 1] - b);
  uint32_t key[kBucketSmall];  // color << 28 | position << 24 ... packed with the id below
  int u[kBucketSmall];
#pragma unroll
  for (int j = 0; j < kBucketSmall; ++j) u[j] = j < d ? __ldg(col + b + j) : 0;
#pragma unroll
  for (int j = 0; j < kBucketSmall; ++j) key[j] = j < d ? (static_cast<uint32_t>(rot_key(colors[u[j]], cv, k)) << 4 | j) : 0xFFFFu;
  // Batcher odd-even merge sort network for 8 keys
#define TCG_CX(a, b) { const uint32_t x = min(key[a], key[b]), y = max(key[a], key[b]); key[a] = x; key[b] = y; }
  TCG_CX(0, 1) TCG_CX(2, 3) TCG_CX(4, 5) TCG_CX(6, 7)
  TCG_CX(0, 2) TCG_CX(1, 3) TCG_CX(4, 6) TCG_CX(5, 7)
  TCG_CX(1, 2) TCG_CX(5, 6)
  TCG_CX(0, 4) TCG_CX(1, 5) TCG_CX(2, 6) TCG_CX(3, 7)
  TCG_CX(2, 4) TCG_CX(3, 5)
  TCG_CX(1, 2) TCG_CX(3, 4) TCG_CX(5, 6)
#undef TCG_CX
#pragma unroll
  for (int j = 0; j < kBucketSmall; ++j) {
    if (j < d) {
      const int pos = static_cast<int>(key[j] & 15);
      int uu = u[0];  // u[pos] with static register indices
#pragma unroll
      for (int q = 1; q < kBucketSmall; ++q) uu = pos == q ? u[q] : uu;
      out[b + j] = pack_entry(static_cast<uint32_t>(uu), static_cast<uint32_t>(unrot_key(static_cast<int>(key[j] >> 4), cv, k)));
    }
  }
  auto below = [&](int c) {  // entries of color < c
    int x = 0;
#pragma unroll
    for (int j = 0; j < kBucketSmall; ++j) x += (j < d) && static_cast<int>(key[j] >> 4) < c;
    return x;
  };
  if (hist)
    for (int c = 0; c < hzw; ++c) {
      const int r = c < k ? rot_key(c, cv, k) : 0;
      hist[static_cast<int64_t>(v) * hzw + c] = c < k ? static_cast<float>(below(r + 1) - below(r)) : 0.f;
    }
  for (int part = 0; part <= nparts; ++part)  // the last cut stops before the own-color run
    cuts[static_cast<int64_t>(v) * (nparts + 1) + part] = b + below(min(part * k / nparts, k - 1));
}

// Rows longer than kBucketLong are cut into chunks of <= kLongChunk entries,
// one CTA each, so a hub row (cfg2: 64K neighbours) is spread over many SMs.
// chunk = {row, begin, end (offsets within the row), chunk index within the
// row}.  Three passes:
// per-chunk color counts, a per-row scan (color-major, chunk order: stable),
// and the scatter (warp w of a chunk owns its w-th contiguous slice).
constexpr int kLongChunk = 4096;

// per-warp color counts of this CTA's chunk slice into cnt[8][k] (smem)
__device__ __forceinline__ void long_chunk_counts(const int32_t* __restrict__ col, const uint8_t* __restrict__ colors,
                                                  int64_t sb, int64_t se, int* cnt, int cv, int k) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t j = sb; j < se; j += 32) {
    const bool ok = j + lane < se;
    const int key = ok ? rot_key(colors[col[j + lane]], cv, k) : -1;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    if (ok && (same & lt) == 0) cnt[key] += __popc(same);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256)
bucket_long_count(const int4* __restrict__ chunks, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                  const uint8_t* __restrict__ colors, const uint8_t* __restrict__ rowc, int k, int* __restrict__ ccnt) {
  __shared__ int wc[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 ch = chunks[blockIdx.x];
  wc[warp][lane] = 0;
  __syncwarp();
  const int64_t rb = row_ptr[ch.x];
  const int64_t slice = (kLongChunk / 8);
  const int64_t sb = min(rb + ch.z, rb + ch.y + warp * slice);
  const int64_t se = min(rb + ch.z, sb + slice);
  long_chunk_counts(col, colors, sb, se, wc[warp], rowc[ch.x], k);
  __syncthreads();
  if (threadIdx.x < k) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += wc[w][threadIdx.x];
    ccnt[static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x] = t;
  }
}

// warp per long row: lane c = color; per-chunk offsets (in place), histogram, cuts
__global__ void __launch_bounds__(256)
bucket_long_scan(const int4* __restrict__ chunks, const int32_t* __restrict__ row_first_chunk, const int64_t* __restrict__ row_ptr,
                 const uint8_t* __restrict__ rowc, int nlong, int k, int nparts, int* __restrict__ ccnt, int64_t* __restrict__ cuts,
                 float* __restrict__ hist, int hzw) {
  const int lane = threadIdx.x & 31;
  const int r = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  if (r >= nlong) return;
  const int c0 = row_first_chunk[r], c1 = row_first_chunk[r + 1];
  const int32_t v = chunks[c0].x;
  const int64_t b = row_ptr[v];
  int tot = 0;
  if (lane < k)
    for (int c = c0; c < c1; ++c) tot += ccnt[static_cast<int64_t>(c) * 32 + lane];
  const int cv = rowc[v];  // lane = rotated key; its color's histogram entry
  if (hist && lane < k) hist[static_cast<int64_t>(v) * hzw + unrot_key(lane, cv, k)] = static_cast<float>(tot);
  if (hist && lane >= k && lane < hzw) hist[static_cast<int64_t>(v) * hzw + lane] = 0.f;
  int incl = tot;  // exclusive scan over colors
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int base = incl - tot;
  for (int part = 0; part <= nparts; ++part) {
    const int cb = part * k / nparts;
    const int at = __shfl_sync(0xffffffffu, base, cb < k ? cb : k - 1);  // (before the own-color run)
    if (lane == 0) cuts[static_cast<int64_t>(v) * (nparts + 1) + part] = b + at;
  }
  if (lane < k) {
    int run = base;
    for (int c = c0; c < c1; ++c) {
      const int x = ccnt[static_cast<int64_t>(c) * 32 + lane];
      ccnt[static_cast<int64_t>(c) * 32 + lane] = run;
      run += x;
    }
  }
}

__global__ void __launch_bounds__(256)
bucket_long_scatter(const int4* __restrict__ chunks, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    const uint8_t* __restrict__ colors, const uint8_t* __restrict__ rowc, int k, const int* __restrict__ ccnt,
                    uint32_t* __restrict__ out) {
  __shared__ int wc[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int4 ch = chunks[blockIdx.x];
  wc[warp][lane] = 0;
  __syncwarp();
  const int64_t rb = row_ptr[ch.x];
  const int64_t slice = (kLongChunk / 8);
  const int64_t sb = min(rb + ch.z, rb + ch.y + warp * slice);
  const int64_t se = min(rb + ch.z, sb + slice);
  const int cv = rowc[ch.x];
  long_chunk_counts(col, colors, sb, se, wc[warp], cv, k);
  __syncthreads();
  if (threadIdx.x < k) {  // warp-major prefix per color + the chunk's row offset
    int run = ccnt[static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x];
    for (int w = 0; w < 8; ++w) {
      const int x = wc[w][threadIdx.x];
      wc[w][threadIdx.x] = run;
      run += x;
    }
  }
  __syncthreads();
  int* cnt = wc[warp];
  for (int64_t j = sb; j < se; j += 32) {
    const bool ok = j + lane < se;
    const int u = ok ? col[j + lane] : 0;
    const int key = ok ? rot_key(colors[u], cv, k) : -1;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    const int slot = ok ? cnt[key] + __popc(same & lt) : 0;
    __syncwarp();
    if (ok) {
      out[rb + slot] = pack_entry(static_cast<uint32_t>(u), static_cast<uint32_t>(unrot_key(key, cv, k)));
      if ((same & lt) == 0) cnt[key] += __popc(same);
    }
    __syncwarp();
  }
}

// Full table M (C columns) -> compressed table (groups * zw columns): slot t
// of group g of vertex u holds M[u, slot_col[color(u)][g][t]] (0 if unused).
// A CTA stages the full rows of `vpb` vertices in smem (coalesced 128 B panel
// rows), then writes the compressed rows group-major (coalesced as well).
__global__ void __launch_bounds__(256)
rooted_compress(const float* __restrict__ M, int C, const uint8_t* __restrict__ colors,
                const int32_t* __restrict__ slot_col, int groups, int zw, int32_t n, int vpb,
                float* __restrict__ out) {
  extern __shared__ float crow[];
  const int panels = num_panels(C);
  const int zl = last_panel_width(C);
  const int rf = (panels - 1) * kZ + zl;  // floats of one panel-padded row
  const int per = rf / 4;
  const int64_t u0 = static_cast<int64_t>(blockIdx.x) * vpb;
  for (int f = threadIdx.x; f < vpb * per; f += blockDim.x) {
    const int r = f / per, c4 = (f % per) * 4;
    const int64_t u = u0 + r;
    if (u >= n) continue;
    const int p = c4 / kZ, z = c4 % kZ;
    const int zp = p == panels - 1 ? zl : kZ;
    *reinterpret_cast<float4*>(crow + r * rf + c4) =
        __ldg(reinterpret_cast<const float4*>(M + static_cast<int64_t>(p) * n * kZ + u * zp + z));
  }
  __syncthreads();
  const int total = vpb * groups * zw;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int t = i % zw, it = i / zw;
    const int g = it / vpb, r = it % vpb;
    const int64_t u = u0 + r;
    if (u >= n) continue;
    const int col = __ldg(slot_col + (static_cast<int64_t>(colors[u]) * groups + g) * zw + t);
    out[static_cast<int64_t>(g) * n * kZ + u * zw + t] = col >= 0 ? crow[r * rf + col] : 0.f;
  }
}

// One launch = one (group, part).  Task = one segment (lane group of G = ZW/4
// lanes, float4 per lane), as spmm_part.  A ROUND takes the next (up to) R
// entries of the segment that share the first one's color -- rows are color
// sorted, so that is a prefix -- gathers them, and adds their fp32 tree sum
// to the fp64 run accumulator; a color change scatters the run into the
// task's F_g accumulators (smem, fp32: each F_g column receives at most one
// run per color of its set).  The next round's entries are fetched while the
// current round's gathers are in flight (its start only depends on the
// entries' colors).  slot_acc: [K + 1][stride], this group's zw slots at
// offset 0, unused slots (and the whole extra row K, the state before the
// first run) pointing at the dummy accumulator fpad, so the run scatter is
// branch-free; a lane group's accumulators are fpad + 4 floats apart.
// PAIR (pair layout, host.hpp): the row's color cv picks the source copy
// X + cv * xstride, whose slots are indexed by the neighbour color relabeled
// past cv (slot_acc: [k-1][stride]); P' is stored relative to cv as well.
template <int ZW, int MINB, bool PAIR>
__global__ void __launch_bounds__(kSpmmWarps * 32, MINB)
spmm_rooted(const Seg* __restrict__ segs, int64_t ntasks, const uint32_t* __restrict__ colb,
            const int64_t* __restrict__ cuts, int nparts, int part, const int32_t* __restrict__ slot_row,
            const float* __restrict__ X, const int16_t* __restrict__ slot_acc, int slot_stride,
            int fbase, int fpad, int Cstore, int32_t n, float* __restrict__ Y,
            double* __restrict__ partial, int first, const uint8_t* __restrict__ rowc, int64_t xstride, int kdummy) {
  constexpr int G = ZW / 4, SPW = 32 / G, R = 8, NI = R / G;
  extern __shared__ float racc_sm[];
  const int lane = threadIdx.x & 31, g = lane / G, l = lane % G, warp = threadIdx.x >> 5;
  // this group's slot table (K + 1 rows of ZW) after the accumulators
  int16_t* slot_sm = reinterpret_cast<int16_t*>(racc_sm + kSpmmWarps * SPW * (fpad + 4));
  for (int i = threadIdx.x; i < (kdummy + 1) * ZW; i += blockDim.x)
    slot_sm[i] = slot_acc[static_cast<int64_t>(i / ZW) * slot_stride + i % ZW];
  __syncthreads();
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kSpmmWarps + warp;
  if (task >= ntasks) return;
  const Seg s = segs[task * SPW + g];
  float* acc = racc_sm + (warp * SPW + g) * (fpad + 4);
  for (int i = l; i < fpad; i += G) acc[i] = 0.f;
  const uint64_t pstream = policy_evict_first(), pkeep = policy_evict_last();
  // this part's color class of the segment's row: [cut_p, cut_p+1) ∩ segment
  int64_t lo = s.e_begin, hi = s.e_begin;
  uint32_t cv = 0;
  if (s.dst != kSkip) {
    const int32_t row = s.dst >= 0 ? s.dst : slot_row[-1 - s.dst];
    if (PAIR) cv = rowc[row];
    const int64_t* ct = cuts + static_cast<int64_t>(row) * (nparts + 1) + part;
    lo = max(s.e_begin, ct[0]);
    hi = min(s.e_begin + s.len, ct[1]);
    if (hi < lo) hi = lo;
  }
  const uint32_t* cp = colb + lo;
  const int len = static_cast<int>(hi - lo);
  double r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  int cur = kdummy;
  int pos = 0;  // first unconsumed entry of the segment
  auto fetch = [&](int at, uint32_t (&w)[NI]) {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int e = at + i * G + l;
      w[i] = e < len ? static_cast<uint32_t>(ld_stream_i32(reinterpret_cast<const int32_t*>(cp + e), pstream))
                     : kPackSentinel;
    }
  };
  uint32_t w[NI];
  fetch(0, w);
  __syncwarp();
  const char* Xl = reinterpret_cast<const char*>(X + (PAIR ? static_cast<int64_t>(cv) * xstride : 0) + l * 4);
  const int16_t* sla = slot_sm + l * 4;
  auto scatter = [&]() {  // the finished run into its slots' accumulators (dummy for unused slots)
    const short4 sl = *reinterpret_cast<const short4*>(sla + cur * ZW);
    acc[sl.x] += static_cast<float>(r0);
    acc[sl.y] += static_cast<float>(r1);
    acc[sl.z] += static_cast<float>(r2);
    acc[sl.w] += static_cast<float>(r3);
    r0 = r1 = r2 = r3 = 0;
  };
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (g * G);
  for (;;) {
    // the round = the prefix of the next R entries sharing entry 0's color
    // (entry j sits in lane j % G, word j / G of the group)
    const uint32_t c_round = __shfl_sync(0xffffffffu, w[0], 0, G) & kColorMask;
    // the slot table's color index: relabeled past cv in the pair layout
    const uint32_t c_slot = PAIR ? c_round - (c_round > cv ? 1u : 0u) : c_round;
    int count = 0;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const bool ok = w[i] != kPackSentinel && (w[i] & kColorMask) == c_round;
      count += __popc(__ballot_sync(0xffffffffu, ok) & gmask);
    }
    if (!__any_sync(0xffffffffu, count > 0)) break;
    uint32_t pk[R];
#pragma unroll
    for (int j = 0; j < R; ++j) pk[j] = __shfl_sync(0xffffffffu, w[j / G], j % G, G);
    pos += count;
    fetch(pos, w);  // next round's entries, overlapping this round's gathers
    float4 v[R];
    const char* Xr = Xl - c_round * (ZW / 8);  // entry * ZW / 8 = u * ZW * 4 + c_round * ZW / 8
#pragma unroll
    for (int j = 0; j < R; ++j) {
      v[j] = make_float4(0, 0, 0, 0);
      if (j < count) v[j] = ld_keep_f4(row_addr(Xr, pk[j], ZW / 8), pkeep);
    }
    if (count > 0 && static_cast<int>(c_slot) != cur) {
      scatter();
      cur = static_cast<int>(c_slot);
    }
#pragma unroll
    for (int wd = R / 2; wd; wd >>= 1)
#pragma unroll
      for (int j = 0; j < wd; ++j) {
        v[j].x += v[j + wd].x; v[j].y += v[j + wd].y; v[j].z += v[j + wd].z; v[j].w += v[j + wd].w;
      }
    r0 += v[0].x; r1 += v[0].y; r2 += v[0].z; r3 += v[0].w;
  }
  scatter();
  __syncwarp();
  if (s.dst == kSkip) return;
  if (s.dst >= 0) {
    for (int i = l * 4; i < fpad; i += G * 4) {
      const int colc = fbase + i;
      const int p = colc / kZ, z = colc % kZ;
      float* yp = Y + static_cast<int64_t>(p) * n * kZ + static_cast<int64_t>(s.dst) * panel_width(Cstore, p) + z;
      float4 a = *reinterpret_cast<const float4*>(acc + i);
      if (!first) {
        const float4 o = ld_stream_f4(yp, pstream);
        a.x += o.x; a.y += o.y; a.z += o.z; a.w += o.w;
      }
      st_stream_f4(yp, a, pstream);
    }
  } else {
    double* pp = partial + static_cast<int64_t>(-1 - s.dst) * fpad;
    for (int i = l; i < fpad; i += G) pp[i] = acc[i];
  }
}

// Split rows of the rooted SpMM: storage columns [fbase, fbase + fpad) of row
// rows[r] (+)= the sum of the row's fp64 partial slots, in slot order.
__global__ void rooted_fixup(const int32_t* __restrict__ rows, const int32_t* __restrict__ slot_begin,
                             int nrows, const double* __restrict__ partial, int fbase, int fpad, int Cstore,
                             int32_t n, float* __restrict__ Y, int first) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(nrows) * fpad) return;
  const int a = static_cast<int>(i % fpad);
  const int r = static_cast<int>(i / fpad);
  double acc = 0;
  for (int s = slot_begin[r]; s < slot_begin[r + 1]; ++s) acc += partial[static_cast<int64_t>(s) * fpad + a];
  float* y = Y + panel_offset(Cstore, n, rows[r], fbase + a);
  *y = static_cast<float>(first ? acc : acc + static_cast<double>(*y));
}

// Pair layout (host.hpp PairLayout): the passive table M_p, stored RR (column
// j = relabeled index of S minus c(u) over the other k-1 colors), is expanded
// into one copy per row color cv != c(u): copy (cv, l) of vertex u holds, in
// slot order, M_p[u, S] for the sets S of pair group l (sets over the k-1
// colors other than cv) that contain c(u).  A CTA stages the RR rows of 32
// consecutive vertices, then writes each copy's 32 rows (zw floats each) as
// one contiguous block.  xmap: [c(u)][cv][L * zw] -> RR column, or -1.
__global__ void __launch_bounds__(256)
pair_expand(const float* __restrict__ M, int Wx, const uint8_t* __restrict__ colors, const int16_t* __restrict__ xmap,
            int k, int L, int zw, int32_t n, float* __restrict__ out) {
  extern __shared__ float xrow[];  // [32][Wx + 1]
  __shared__ uint8_t cu_s[32];
  const int64_t u0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int pitch = Wx + 1;
  if (threadIdx.x < 32) cu_s[threadIdx.x] = u0 + threadIdx.x < n ? colors[u0 + threadIdx.x] : 0;
  // stage: panel p of the RR table holds the tile's 32 rows contiguously
  const int panels = num_panels(Wx);
  for (int p = 0; p < panels; ++p) {
    const int zp = panel_width(Wx, p);
    const float* src = M + static_cast<int64_t>(p) * n * kZ + u0 * zp;
    for (int f = threadIdx.x; f < 32 * zp / 4; f += blockDim.x) {
      const int r = (f * 4) / zp, c4 = (f * 4) % zp;
      if (u0 + r >= n) continue;
      const float4 x = __ldg(reinterpret_cast<const float4*>(src + static_cast<int64_t>(r) * zp + c4));
      const int c0 = p * kZ + c4;  // (the last panel may be wider than its columns)
      float* d = xrow + r * pitch + c0;
      if (c0 < Wx) d[0] = x.x;
      if (c0 + 1 < Wx) d[1] = x.y;
      if (c0 + 2 < Wx) d[2] = x.z;
      if (c0 + 3 < Wx) d[3] = x.w;
    }
  }
  __syncthreads();
  // copy q = cv * L + l of vertex u0 + r: xmap block (cu * k * L + q), output
  // block q; thread = (r, float4 j) of a copy block, copies strided by qstep
  const int per = 32 * zw / 4;  // float4s of one copy's tile block (64, 128 or 256)
  const int qstep = blockDim.x / per;
  const int f = threadIdx.x % per;
  const int r = f / (zw / 4), j = (f % (zw / 4)) * 4;
  const int64_t u = u0 + r;
  if (u >= n) return;
  const int cu = cu_s[r];
  const float* xr = xrow + r * pitch;
  const int QL = k * L;
  const int16_t* xm = xmap + static_cast<int64_t>(cu) * QL * zw + j;
  float* o = out + u * zw + j;
  for (int q = threadIdx.x / per; q < QL; q += qstep) {
    if (static_cast<unsigned>(q - cu * L) < static_cast<unsigned>(L)) continue;  // cv == cu: never read
    const short4 m = __ldg(reinterpret_cast<const short4*>(xm + q * zw));
    const float4 val = make_float4(m.x >= 0 ? xr[m.x] : 0.f, m.y >= 0 ? xr[m.y] : 0.f, m.z >= 0 ? xr[m.z] : 0.f,
                                   m.w >= 0 ? xr[m.w] : 0.f);
    __stcs(reinterpret_cast<float4*>(o + static_cast<int64_t>(q) * n * zw), val);
  }
}

// Per coloring, the whole-row segment schedule re-ordered by the row's color
// (stable: length order within a color), so that the pair SpMM's rows of one
// color -- which all gather from copy cv -- run together and the copy's
// lines stay in L2.  Key k = padding.
__global__ void seg_keys(const Seg* __restrict__ segs, int64_t nseg, const int32_t* __restrict__ slot_row,
                         const uint8_t* __restrict__ rowc, int k, uint8_t* __restrict__ keys) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nseg) return;
  const Seg s = segs[i];
  keys[i] = s.dst == kSkip ? static_cast<uint8_t>(k) : rowc[s.dst >= 0 ? s.dst : slot_row[-1 - s.dst]];
}
__global__ void seg_gather(const Seg* __restrict__ segs, const int32_t* __restrict__ perm, int64_t nseg,
                           Seg* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nseg) out[i] = segs[perm[i]];
}

// tcg_set_graph on the device: every id in range, no self-loop, rows strictly
// ascending (graph.hpp invariants).  Warp per row; bad = 1 (range / loop) or
// 2 (order), the first writer wins.
__global__ void __launch_bounds__(256)
validate_csr(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int32_t n, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); v < n; v += nwarps) {
    const int64_t b = row_ptr[v], e = row_ptr[v + 1];
    int err = 0;
    for (int64_t j = b + lane; j < e; j += 32) {
      const int32_t u = col[j];
      if (u < 0 || u >= n || u == v) err = 1;
      else if (j > b && col[j - 1] >= u) err = 2;
    }
    if (__any_sync(0xffffffffu, err) && err) atomicCAS(bad, 0, err);
  }
}

// Split rows: Y[row] (+)= sum of the row's fp64 partial slots, in slot order.
__global__ void spmm_fixup(const int32_t* __restrict__ rows, const int32_t* __restrict__ slot_begin,
                           int nrows, const double* __restrict__ partial, float* __restrict__ Y,
                           int zw, int first) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(nrows) * zw) return;
  const int z = static_cast<int>(i % zw);
  const int r = static_cast<int>(i / zw);
  double acc = 0;
  for (int s = slot_begin[r]; s < slot_begin[r + 1]; ++s) acc += partial[static_cast<int64_t>(s) * zw + z];
  float* y = Y + static_cast<int64_t>(rows[r]) * zw + z;
  *y = static_cast<float>(first ? acc : acc + static_cast<double>(*y));
}

// ------------------------------------------------------------------- eMA

// Stage a 32-vertex tile of a panel table into smem, column-major [c][33].
// The tile of every full panel is one contiguous 4 KB block; float4 index f
// over the whole tile maps to (panel, vertex, column quad).  Each thread keeps
// kStageU independent 16 B loads in flight before storing, so staging runs
// at bandwidth rather than at one HBM latency per float4.
template <int kStageU>
__device__ __forceinline__ void stage_tile(const float* __restrict__ T, int C, int32_t n, int64_t v0,
                                           float* dst) {
  const int panels = num_panels(C);
  const int zl = last_panel_width(C);
  const int full4 = (panels - 1) * kTileV * (kZ / 4);   // float4s in full panels
  const int total4 = full4 + kTileV * (zl / 4);
  for (int base = threadIdx.x; base < total4; base += blockDim.x * kStageU) {
    float4 x[kStageU];
    int c0[kStageU], vv[kStageU];
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int f = base + u * blockDim.x;
      int p, r, zw;
      if (f < full4) { p = f / (kTileV * 8); r = f % (kTileV * 8); zw = kZ; }
      else { p = panels - 1; r = f - full4; zw = zl; }
      const int q4 = zw / 4;
      vv[u] = r / q4;
      c0[u] = p * kZ + (r % q4) * 4;
      x[u] = make_float4(0, 0, 0, 0);
      if (f < total4 && v0 + vv[u] < n)
        x[u] = __ldg(reinterpret_cast<const float4*>(T + static_cast<int64_t>(p) * n * kZ + (v0 + vv[u]) * zw + (r % q4) * 4));
      if (f >= total4) c0[u] = C;  // nothing to store
    }
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int c = c0[u];
      if (c + 0 < C) dst[(c + 0) * kSpitch + vv[u]] = x[u].x;
      if (c + 1 < C) dst[(c + 1) * kSpitch + vv[u]] = x[u].y;
      if (c + 2 < C) dst[(c + 2) * kSpitch + vv[u]] = x[u].z;
      if (c + 3 < C) dst[(c + 3) * kSpitch + vv[u]] = x[u].w;
    }
  }
}

// stage_tile for a P' stored group-major (rooted layout): storage column c
// goes to smem row inv[c] (the combinadic column), padding (-1) is dropped.
// Cstore is a multiple of 8, so a float4 never straddles its end.
template <int kStageU>
__device__ __forceinline__ void stage_tile_map(const float* __restrict__ T, int Cstore, int32_t n, int64_t v0,
                                               float* dst, const int32_t* __restrict__ inv) {
  const int panels = num_panels(Cstore);
  const int zl = last_panel_width(Cstore);
  const int full4 = (panels - 1) * kTileV * (kZ / 4);
  const int total4 = full4 + kTileV * (zl / 4);
  for (int base = threadIdx.x; base < total4; base += blockDim.x * kStageU) {
    float4 x[kStageU];
    int c0[kStageU], vv[kStageU];
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int f = base + u * blockDim.x;
      int p, r, zw;
      if (f < full4) { p = f / (kTileV * 8); r = f % (kTileV * 8); zw = kZ; }
      else { p = panels - 1; r = f - full4; zw = zl; }
      const int q4 = zw / 4;
      vv[u] = r / q4;
      c0[u] = p * kZ + (r % q4) * 4;
      x[u] = make_float4(0, 0, 0, 0);
      if (f < total4 && v0 + vv[u] < n && c0[u] < Cstore)
        x[u] = __ldg(reinterpret_cast<const float4*>(T + static_cast<int64_t>(p) * n * kZ + (v0 + vv[u]) * zw + (r % q4) * 4));
      if (f >= total4) c0[u] = Cstore;
    }
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      if (c0[u] >= Cstore) continue;
      const int4 m = __ldg(reinterpret_cast<const int4*>(inv + c0[u]));
      if (m.x >= 0) dst[m.x * kSpitch + vv[u]] = x[u].x;
      if (m.y >= 0) dst[m.y * kSpitch + vv[u]] = x[u].y;
      if (m.z >= 0) dst[m.z * kSpitch + vv[u]] = x[u].z;
      if (m.w >= 0) dst[m.w * kSpitch + vv[u]] = x[u].w;
    }
  }
}

// Non-root node.  M_s[v,S] = sum_p M_a[v, A(S,p)] * P'[v, P(S,p)] over the
// by-parent split pairs (color_index.hpp:97-98,131-165).  Warp w computes
// chunks of 8 consecutive parent columns (8 independent accumulators) for its
// 32 vertices and writes each 32 B row chunk directly.  ALEAF: M_a is one-hot
// at color(v), so M_s[v,S] = P'[v, S minus color(v)] if color(v) is in S --
// `drop[S*k + c]` holds that column (or -1).
template <bool ALEAF, bool STAGED>
__global__ void __launch_bounds__(kEmaWarps * 32)
ema_node(const float* __restrict__ Am, const float* __restrict__ Pm,
         const uint8_t* __restrict__ colors, const int2* __restrict__ split,
         const uint32_t* __restrict__ packed, const int32_t* __restrict__ drop, int k, int pairs,
         int Ca, int Cp, int Cs, int32_t n, float* __restrict__ out) {
  extern __shared__ float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v0 = static_cast<int64_t>(blockIdx.x) * kTileV;
  const int64_t v = v0 + lane;
  const bool valid = v < n;
  float* sA = smem;
  float* sP = smem + (ALEAF ? 0 : Ca * kSpitch);
  if (STAGED) {
    if (!ALEAF) stage_tile<1>(Am, Ca, n, v0, sA);
    stage_tile<1>(Pm, Cp, n, v0, sP);
    __syncthreads();
  }
  const int my_color = valid ? colors[v] : 0;
  auto pval = [&](int ip) -> float {
    if (STAGED) return sP[ip * kSpitch + lane];
    return valid ? Pm[panel_offset(Cp, n, v, ip)] : 0.f;
  };
  auto aval = [&](int ia) -> float {
    if (STAGED) return sA[ia * kSpitch + lane];
    return valid ? Am[panel_offset(Ca, n, v, ia)] : 0.f;
  };
  const int nchunks = (Cs + 7) / 8;
  for (int q = warp; q < nchunks; q += blockDim.x >> 5) {
    float r[8];
    if (ALEAF) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int S = q * 8 + j;
        const int d = S < Cs ? __ldg(drop + static_cast<int64_t>(S) * k + my_color) : -1;
        r[j] = d >= 0 ? pval(d) : 0.f;
      }
    } else if (packed) {
      // split pairs packed as (I_a | I_p << 16): each lane loads one pair per
      // parent column for a batch of 32 pairs (coalesced), then the pairs are
      // broadcast with shuffles -- no per-pair L1/L2 round trip
      const int nv = min(8, Cs - q * 8);
      const uint32_t* sp = packed + static_cast<int64_t>(q) * 8 * pairs;
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = 0.f;
      for (int pb = 0; pb < pairs; pb += 32) {
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          w[j] = (j < nv && pb + lane < pairs) ? __ldg(sp + j * pairs + pb + lane) : 0u;
        const int cnt = min(32, pairs - pb);
        for (int pp = 0; pp < cnt; ++pp) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t s = __shfl_sync(0xffffffffu, w[j], pp);
            r[j] = fmaf(aval(static_cast<int>(s & 0xFFFFu)), pval(static_cast<int>(s >> 16)), r[j]);
          }
        }
      }
    } else {
      const int nv = min(8, Cs - q * 8);
      const int2* sp = split + static_cast<int64_t>(q) * 8 * pairs;
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = 0.f;
      for (int p = 0; p < pairs; ++p) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < nv) {
            const int2 s = __ldg(sp + j * pairs + p);
            r[j] = fmaf(aval(s.x), pval(s.y), r[j]);
          }
        }
      }
    }
    if (valid) {
      const int c0 = q * 8;
      const int zw = panel_width(Cs, c0 / kZ);
      float* dst = out + static_cast<int64_t>(c0 / kZ) * n * kZ + v * zw + (c0 % kZ);
      reinterpret_cast<float4*>(dst)[0] = make_float4(r[0], r[1], r[2], r[3]);
      if (zw > 4 && (c0 % kZ) + 4 < zw) reinterpret_cast<float4*>(dst)[1] = make_float4(r[4], r[5], r[6], r[7]);
    }
  }
}

// ----------------------------------------------------- register-blocked eMA
// Colors split into H1 = {0..5} and H2 = {6..k-1}.  The combinadic index of a
// set X = X1 u X2 is idx(X1) + g(X2, |X1|) (X1's colors take the low
// positions), so for fixed (X2, |X1|) the columns {X1 u X2} are one
// contiguous range of C(6,|X1|) columns.  The eMA therefore decomposes into
// BLOCKS: an output group (S2, s1) -- C(6,s1) contiguous output columns held
// in registers -- accumulates, for every split of S2 into (a2, p2) and
// (i, j) with i + j = s1, the fixed H1 "micro-pattern" of disjoint (a1, p1)
// pairs over C(6,i) A values and C(6,j) P values loaded once into registers.
// Loads per FMA drop from 2 to ~0.65 on the wide nodes.
constexpr int kH1 = 6;
constexpr int kMaxAcc = 20;  // C(6,3)

__host__ __device__ constexpr int cbin(int a, int b) {
  if (b < 0 || b > a) return 0;
  int r = 1;
  for (int i = 1; i <= b; ++i) r = r * (a - b + i) / i;
  return r;
}
// C(H, s) for a runtime s: H + 1 selects of compile-time constants (no
// integer division in the epilogues)
template <int H>
__device__ __forceinline__ int cbin_rt(int s) {
  int r = 0;
#pragma unroll
  for (int t = 0; t <= H; ++t) r = s == t ? cbin(H, t) : r;
  return r;
}
__host__ __device__ constexpr int cpop(unsigned m) {
  int c = 0;
  for (; m; m &= m - 1) ++c;
  return c;
}
__host__ __device__ constexpr int cidx(unsigned m) {  // combinadic rank of a subset of H1
  int idx = 0, pos = 0;
  for (int c = 0; c < kH1; ++c)
    if (m >> c & 1u) idx += cbin(c, ++pos);
  return idx;
}
struct Trip {
  int a, p, o;
};
// t-th disjoint (a1, p1) pair with |a1| = I, |p1| = J, in a fixed order
__host__ __device__ constexpr Trip nth_trip(int I, int J, int t) {
  int n = 0;
  for (unsigned am = 0; am < (1u << kH1); ++am) {
    if (cpop(am) != I) continue;
    for (unsigned pm = 0; pm < (1u << kH1); ++pm) {
      if (cpop(pm) != J || (am & pm)) continue;
      if (n == t) return Trip{cidx(am), cidx(pm), cidx(am | pm)};
      ++n;
    }
  }
  return Trip{0, 0, 0};
}
template <int I, int J, int T>
struct TripC {
  static constexpr Trip v = nth_trip(I, J, T);
};

template <int I, int J, int... T>
__device__ __forceinline__ void micro_fma(const float (&a)[kMaxAcc], const float (&p)[kMaxAcc],
                                          float (&acc)[kMaxAcc], std::integer_sequence<int, T...>) {
  ((acc[TripC<I, J, T>::v.o] = fmaf(a[TripC<I, J, T>::v.a], p[TripC<I, J, T>::v.p], acc[TripC<I, J, T>::v.o])), ...);
}

template <int I, int J>
__device__ __forceinline__ void micro_block(const float* __restrict__ sa, const float* __restrict__ sp,
                                            float (&acc)[kMaxAcc]) {
  constexpr int NA = cbin(kH1, I), NP = cbin(kH1, J), NT = cbin(kH1, I) * cbin(kH1 - I, J);
  float a[kMaxAcc], p[kMaxAcc];
#pragma unroll
  for (int x = 0; x < NA; ++x) a[x] = sa[x * kSpitch];
#pragma unroll
  for (int x = 0; x < NP; ++x) p[x] = sp[x * kSpitch];
  micro_fma<I, J>(a, p, acc, std::make_integer_sequence<int, NT>{});
}

struct GroupDesc {      // one output group: C(6, s1) contiguous parent columns
  int32_t out_off, s1, b0, b1;
};
struct BlockDesc {      // A range at a_off (|a1| = i), P range at p_off (|p1| = j)
  int32_t a_off, p_off;
  int32_t ij;           // i * 8 + j
  int32_t pad;
};

#define TCG_IJ(I, J) \
  case I * 8 + J: micro_block<I, J>(sA + bd.a_off * kSpitch + lane, sP + bd.p_off * kSpitch + lane, acc); break;

template <bool STAGED>
__global__ void __launch_bounds__(256)
ema_blocked(const float* __restrict__ Am, const float* __restrict__ Pm,
            const GroupDesc* __restrict__ groups, int ngroups, const BlockDesc* __restrict__ blocks,
            int Ca, int Cp, int Cs, int32_t n, float* __restrict__ out, int Cps,
            const int32_t* __restrict__ pinv) {
  extern __shared__ float smem[];
  __shared__ int next_group;
  const int lane = threadIdx.x & 31;
  const int64_t v0 = static_cast<int64_t>(blockIdx.x) * kTileV;
  const int64_t v = v0 + lane;
  float* sA = smem;
  float* sP = smem + Ca * kSpitch;
  if (threadIdx.x == 0) next_group = blockDim.x / 32;
  stage_tile<8>(Am, Ca, n, v0, sA);
  if (pinv) stage_tile_map<8>(Pm, Cps, n, v0, sP, pinv);
  else stage_tile<8>(Pm, Cp, n, v0, sP);
  __syncthreads();
  // groups are sorted by work (descending); warps take them dynamically
  for (int gi = threadIdx.x >> 5; gi < ngroups;) {
    const GroupDesc gd = groups[gi];
    float acc[kMaxAcc];
#pragma unroll
    for (int x = 0; x < kMaxAcc; ++x) acc[x] = 0.f;
    for (int b = gd.b0; b < gd.b1; ++b) {
      const BlockDesc bd = blocks[b];
      switch (bd.ij) {
        TCG_IJ(0, 1) TCG_IJ(0, 2) TCG_IJ(0, 3) TCG_IJ(0, 4) TCG_IJ(0, 5) TCG_IJ(0, 6)
        TCG_IJ(1, 0) TCG_IJ(1, 1) TCG_IJ(1, 2) TCG_IJ(1, 3) TCG_IJ(1, 4) TCG_IJ(1, 5)
        TCG_IJ(2, 0) TCG_IJ(2, 1) TCG_IJ(2, 2) TCG_IJ(2, 3) TCG_IJ(2, 4)
        TCG_IJ(3, 0) TCG_IJ(3, 1) TCG_IJ(3, 2) TCG_IJ(3, 3)
        TCG_IJ(4, 0) TCG_IJ(4, 1) TCG_IJ(4, 2)
        TCG_IJ(5, 0) TCG_IJ(5, 1)
        TCG_IJ(6, 0) TCG_IJ(0, 0)
        default: break;
      }
    }
    if (v < n) {
      const int cnt = cbin_rt<kH1>(gd.s1);
#pragma unroll
      for (int x = 0; x < kMaxAcc; ++x)
        if (x < cnt) out[panel_offset(Cs, n, v, gd.out_off + x)] = acc[x];
    }
    if (lane == 0) gi = atomicAdd(&next_group, 1);
    gi = __shfl_sync(0xffffffffu, gi, 0);
  }
}
#undef TCG_IJ

// ------------------------------------------ vertex-per-CTA eMA (huge nodes)
// When a 32-vertex tile of a node's inputs does not fit in shared memory
// (k = 15/17: a single A row can be 97 KB), a CTA owns ONE vertex at a time:
// its A and P rows are staged contiguously in smem (128 B panel rows, fully
// coalesced loads) and the threads split the node's work -- output groups
// (blocked micro-patterns), parent columns (active leaf) or split pairs (root).
// Persistent grid-stride over vertices; several CTAs per SM overlap staging
// with compute.
// floats of one vertex's panel-padded row (a multiple of 4)
__device__ __forceinline__ int row_floats(int C) { return (num_panels(C) - 1) * kZ + last_panel_width(C); }

__device__ __forceinline__ void stage_row(const float* __restrict__ T, int C, int32_t n, int64_t v,
                                          float* dst) {
  const int panels = num_panels(C);
  const int zl = last_panel_width(C);
  const int total4 = ((panels - 1) * kZ + zl) / 4;
  for (int f = threadIdx.x; f < total4; f += blockDim.x) {
    const int p = (f * 4) / kZ, z4 = (f * 4) % kZ;
    const int zw = p == panels - 1 ? zl : kZ;
    const float4 x = __ldg(reinterpret_cast<const float4*>(T + static_cast<int64_t>(p) * n * kZ + v * zw + z4));
    *reinterpret_cast<float4*>(dst + p * kZ + z4) = x;
  }
}

// stage_row of a group-major P' (see stage_tile_map): dst[inv[c]] = row[c]
__device__ __forceinline__ void stage_row_map(const float* __restrict__ T, int Cstore, int32_t n, int64_t v,
                                              float* dst, const int32_t* __restrict__ inv) {
  const int panels = num_panels(Cstore);
  const int zl = last_panel_width(Cstore);
  const int total4 = Cstore / 4;
  for (int f = threadIdx.x; f < total4; f += blockDim.x) {
    const int p = (f * 4) / kZ, z4 = (f * 4) % kZ;
    const int zw = p == panels - 1 ? zl : kZ;
    const float4 x = __ldg(reinterpret_cast<const float4*>(T + static_cast<int64_t>(p) * n * kZ + v * zw + z4));
    const int4 m = __ldg(reinterpret_cast<const int4*>(inv + f * 4));
    if (m.x >= 0) dst[m.x] = x.x;
    if (m.y >= 0) dst[m.y] = x.y;
    if (m.z >= 0) dst[m.z] = x.z;
    if (m.w >= 0) dst[m.w] = x.w;
  }
}

#define TCG_IJV(I, J) \
  case I * 8 + J: micro_block_v<I, J>(sA + bd.x, sP + bd.y, acc); break;

template <int I, int J>
__device__ __forceinline__ void micro_block_v(const float* __restrict__ sa, const float* __restrict__ sp,
                                              float (&acc)[kMaxAcc]) {
  constexpr int NA = cbin(kH1, I), NP = cbin(kH1, J), NT = cbin(kH1, I) * cbin(kH1 - I, J);
  float a[kMaxAcc], p[kMaxAcc];
#pragma unroll
  for (int x = 0; x < NA; ++x) a[x] = sa[x];
#pragma unroll
  for (int x = 0; x < NP; ++x) p[x] = sp[x];
  micro_fma<I, J>(a, p, acc, std::make_integer_sequence<int, NT>{});
}

// groups: GroupDesc list (sorted by work); blocks: BlockDesc list.  Thread t
// takes groups in a snake order over the threads (balanced, deterministic).
__global__ void __launch_bounds__(256)
ema_vtx_blocked(const float* __restrict__ Am, const float* __restrict__ Pm,
                const GroupDesc* __restrict__ groups, int ngroups, const BlockDesc* __restrict__ blocks,
                int Ca, int Cp, int Cs, int32_t n, float* __restrict__ out, int Cps,
                const int32_t* __restrict__ pinv) {
  extern __shared__ float smem[];
  float* sA = smem;
  float* sP = smem + row_floats(Ca);  // stage_row writes the panel-padded row
  const int T = blockDim.x;
  for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
    __syncthreads();
    stage_row(Am, Ca, n, v, sA);
    if (pinv) stage_row_map(Pm, Cps, n, v, sP, pinv);
    else stage_row(Pm, Cp, n, v, sP);
    __syncthreads();
    for (int r = 0;; ++r) {
      const int gi = (r & 1) ? (r + 1) * T - 1 - static_cast<int>(threadIdx.x) : r * T + static_cast<int>(threadIdx.x);
      if (r * T >= ngroups) break;
      if (gi >= ngroups) continue;
      const GroupDesc gd = groups[gi];
      float acc[kMaxAcc];
#pragma unroll
      for (int x = 0; x < kMaxAcc; ++x) acc[x] = 0.f;
      for (int b = gd.b0; b < gd.b1; ++b) {
        const BlockDesc b4 = blocks[b];
        const int2 bd = make_int2(b4.a_off, b4.p_off);
        switch (b4.ij) {
          TCG_IJV(0, 1) TCG_IJV(0, 2) TCG_IJV(0, 3) TCG_IJV(0, 4) TCG_IJV(0, 5) TCG_IJV(0, 6)
          TCG_IJV(1, 0) TCG_IJV(1, 1) TCG_IJV(1, 2) TCG_IJV(1, 3) TCG_IJV(1, 4) TCG_IJV(1, 5)
          TCG_IJV(2, 0) TCG_IJV(2, 1) TCG_IJV(2, 2) TCG_IJV(2, 3) TCG_IJV(2, 4)
          TCG_IJV(3, 0) TCG_IJV(3, 1) TCG_IJV(3, 2) TCG_IJV(3, 3)
          TCG_IJV(4, 0) TCG_IJV(4, 1) TCG_IJV(4, 2)
          TCG_IJV(5, 0) TCG_IJV(5, 1)
          TCG_IJV(6, 0) TCG_IJV(0, 0)
          default: break;
        }
      }
      const int cnt = cbin_rt<kH1>(gd.s1);
#pragma unroll
      for (int x = 0; x < kMaxAcc; ++x)
        if (x < cnt) out[panel_offset(Cs, n, v, gd.out_off + x)] = acc[x];
    }
  }
}
#undef TCG_IJV

// Active leaf, one vertex per CTA: M_s[v,S] = P'[v, S minus color(v)] or 0.
__global__ void __launch_bounds__(256)
ema_vtx_aleaf(const float* __restrict__ Pm, const uint8_t* __restrict__ colors,
              const int32_t* __restrict__ drop, int k, int Cp, int Cs, int32_t n, float* __restrict__ out) {
  extern __shared__ float smem[];
  for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
    __syncthreads();
    stage_row(Pm, Cp, n, v, smem);
    __syncthreads();
    const int c = colors[v];
    const int panels = num_panels(Cs);
    // write the row panel by panel, float4 per thread (coalesced 128 B rows)
    const int zl = last_panel_width(Cs);
    const int total4 = ((panels - 1) * kZ + zl) / 4;
    for (int f = threadIdx.x; f < total4; f += blockDim.x) {
      const int p = (f * 4) / kZ, z4 = (f * 4) % kZ;
      const int zw = p == panels - 1 ? zl : kZ;
      float r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int S = p * kZ + z4 + j;
        const int d = S < Cs ? __ldg(drop + static_cast<int64_t>(S) * k + c) : -1;
        r[j] = d >= 0 ? smem[d] : 0.f;
      }
      *reinterpret_cast<float4*>(out + static_cast<int64_t>(p) * n * kZ + v * zw + z4) = make_float4(r[0], r[1], r[2], r[3]);
    }
  }
}

// Root, one vertex per CTA: fp64 dot product over the split pairs, fixed-order
// block reduction; root_out[v] (the tile totals are then reduced by root_reduce
// over root_out itself).
__global__ void __launch_bounds__(256)
ema_vtx_root(const float* __restrict__ Am, const float* __restrict__ Pm, const uint8_t* __restrict__ colors,
             const int2* __restrict__ split, int pairs, int Ca, int Cp, int aleaf, int32_t n,
             double* __restrict__ root_out, double* __restrict__ root_acc) {
  extern __shared__ float smem[];
  __shared__ double red[256];
  float* sA = smem;
  float* sP = smem + (aleaf ? 0 : row_floats(Ca));
  for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
    __syncthreads();
    if (!aleaf) stage_row(Am, Ca, n, v, sA);
    stage_row(Pm, Cp, n, v, sP);
    __syncthreads();
    const int c = colors[v];
    double acc = 0;
    for (int p = threadIdx.x; p < pairs; p += blockDim.x) {
      const int2 s = __ldg(split + p);
      const float a = aleaf ? (s.x == c ? 1.f : 0.f) : sA[s.x];
      acc = fma(static_cast<double>(a), static_cast<double>(sP[s.y]), acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      root_out[v] = red[0];
      if (root_acc) root_acc[v] += red[0];
    }
  }
}

// Root node: one parent column; warps split the pair list, fp64 throughout,
// fixed-order reduction; per-vertex counts (fp64) and per-tile totals.
template <bool ALEAF, bool STAGED>
__global__ void __launch_bounds__(kEmaWarps * 32)
ema_root(const float* __restrict__ Am, const float* __restrict__ Pm,
         const uint8_t* __restrict__ colors, const int2* __restrict__ split, int pairs, int Ca,
         int Cp, int32_t n, double* __restrict__ root_out, double* __restrict__ root_acc,
         double* __restrict__ tile_tot) {
  extern __shared__ float smem[];
  __shared__ double red[kEmaWarps][kTileV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t v0 = static_cast<int64_t>(blockIdx.x) * kTileV;
  const int64_t v = v0 + lane;
  const bool valid = v < n;
  float* sA = smem;
  float* sP = smem + (ALEAF ? 0 : Ca * kSpitch);
  if (STAGED) {
    if (!ALEAF) stage_tile<1>(Am, Ca, n, v0, sA);
    stage_tile<1>(Pm, Cp, n, v0, sP);
    __syncthreads();
  }
  const int my_color = valid ? colors[v] : -1;
  double acc = 0;
  for (int p = warp; p < pairs; p += kEmaWarps) {
    const int2 s = __ldg(split + p);
    const float a = ALEAF ? (s.x == my_color ? 1.f : 0.f)
                          : (STAGED ? sA[s.x * kSpitch + lane] : (valid ? Am[panel_offset(Ca, n, v, s.x)] : 0.f));
    const float pv = STAGED ? sP[s.y * kSpitch + lane] : (valid ? Pm[panel_offset(Cp, n, v, s.y)] : 0.f);
    acc = fma(static_cast<double>(a), static_cast<double>(pv), acc);
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    double tot = 0;
    for (int w = 0; w < kEmaWarps; ++w) tot += red[w][lane];
    if (valid) {
      root_out[v] = tot;
      if (root_acc) root_acc[v] += tot;
    } else {
      tot = 0;
    }
    for (int o = 16; o; o >>= 1) tot += __shfl_down_sync(0xffffffffu, tot, o);
    if (lane == 0) tile_tot[blockIdx.x] = tot;
  }
}

// Deterministic fp64 sum of the per-tile totals (engines.hpp:125-129; the
// reference's sequential sum differs only at the 1e-16 level).
// Per-vertex root counts (internal row order) of segment s (len values each;
// one segment per copy of a batch) -> total[s], in a fixed shape that only
// depends on len -- so a coloring's total does not depend on whether it ran
// alone or as one copy of a batch: CTA (s, c) of kRootChunks sums its
// contiguous chunk (256 strided partials + a halving tree) into part[], then
// root_reduce folds the kRootChunks partials of each segment in order.
constexpr int kRootChunks = 64;
__global__ void __launch_bounds__(256)
root_partial(const double* __restrict__ x, int64_t len, double* __restrict__ part) {
  __shared__ double red[256];
  const int64_t seg = blockIdx.x / kRootChunks, c = blockIdx.x % kRootChunks;
  const int64_t b = len * c / kRootChunks, e = len * (c + 1) / kRootChunks;
  const double* xs = x + seg * len;
  double s = 0;
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) s += xs[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void root_reduce(const double* __restrict__ x, int64_t len,
                            double* __restrict__ total) {
  __shared__ double red[1024];
  const double* tile_tot = x + static_cast<int64_t>(blockIdx.x) * len;
  total += blockIdx.x;
  double s = 0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) s += tile_tot[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = red[0];
}

// --------------------------------------------------- batched colorings
// Colorings on a batch axis: B colorings of a small graph run
// as ONE coloring of the B-fold disjoint union (copy b = rows [b n, (b+1) n)),
// so every launch of the DP covers B colorings.
__global__ void union_graph(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int32_t n,
                            int64_t nnz, int B, int64_t* __restrict__ rpU, int32_t* __restrict__ colU) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t t = t0; t <= static_cast<int64_t>(n) * B; t += stride)
    rpU[t] = t == static_cast<int64_t>(n) * B ? nnz * B : (t / n) * nnz + rp[t % n];
  for (int64_t t = t0; t < nnz * B; t += stride)
    colU[t] = static_cast<int32_t>((t / nnz) * n + col[t % nnz]);
}
// colors of copy b = coloring b, in internal row order
__global__ void batch_colors(const uint8_t* __restrict__ in, int64_t nglob, const int32_t* __restrict__ perm,
                             int32_t n, int B, uint8_t* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(n) * B) return;
  const int64_t b = t / n, i = t % n;
  out[t] = in[b * nglob + (perm ? perm[i] : i)];
}
// per-vertex accumulation over the copies in coloring order (== one
// root_acc[v] += count per coloring)
__global__ void fold_copies(const double* __restrict__ pv, int32_t n, int B, double* __restrict__ acc) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = acc[i];
  for (int b = 0; b < B; ++b) s += pv[static_cast<int64_t>(b) * n + i];
  acc[i] = s;
}

}  // namespace dev
}  // namespace tcg
