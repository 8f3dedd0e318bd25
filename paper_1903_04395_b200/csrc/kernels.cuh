// kernels.cuh -- the sm_100a kernels of one coloring (SURVEY 2.1 kernel inventory).
//
// Count tables live in HBM as fp32 PANELS: a table with C color-set columns
// is ceil(C/Z) panels, each n x Z floats vertex-major, Z = 16 (64 B per
// vertex per panel = two 32 B sectors).  One panel of an n = 2^20 table is
// 64 MB, so the SpMM's gather source stays resident in the 126 MB L2 while
// every SM sweeps the same panel (measured: 64 B gathers from a 64 MB
// footprint run at ~15.5 TB/s vs ~2.9 TB/s once the footprint spills;
// tools/microbench, profiles/r01_membench.txt).
//
//   mt_coloring   random_coloring (count_table.hpp:90-99): MT19937-64,
//                 one CTA per seed, rejection handled by a block scan
//   nbr_hist      SpMM against a LEAF passive table (one-hot colors,
//                 count_table.hpp:102-107): per-vertex neighbour color
//                 histogram read from 1-byte colors
//   spmm_panels   SpMM of the CSR adjacency against an internal passive
//                 table (la_kernels.hpp:83-102): 4-lane groups gather 64 B
//                 row panels, fp64 accumulation, long rows split into
//                 segments with a deterministic fix-up
//   ema_tile      fused eMA color-set combine (engines.hpp:252-268 +
//                 la_kernels.hpp:106-114) by parent column: 32-vertex tiles
//                 staged in smem, lane = vertex, split pairs warp-uniform;
//                 active-leaf / root (fp64) variants
//   root_reduce   deterministic fp64 total (engines.hpp:125-129)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "layout.hpp"

namespace tcg {
namespace dev {

// ------------------------------------------------------------ load helpers
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ld_stream_i32(const int32_t* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ld_keep_f4(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream_f4(float* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// ------------------------------------------------------------ MT19937-64
// Exactly std::mt19937_64 ([rand.predef]; libstdc++ _M_gen_rand) feeding
// Rng::below (rng.hpp:21-27).  One CTA per seed.  Each 312-word twist runs
// in two dependent phases on 156 threads (words 0..155 read only old state;
// word 156+t reads new word t, which thread t itself produced; word 311
// reads new words 0 and 155), then every word is tempered, tested against
// the rejection threshold and reduced mod k in parallel.  Accepted words map
// to consecutive vertices through a block-wide exclusive scan of the
// rejection flags, so any number of rejections is handled exactly.
constexpr int kMtThreads = 160;

__global__ void __launch_bounds__(kMtThreads)
mt_coloring(const uint64_t* __restrict__ seeds, int32_t n, int k, uint64_t limit,
            uint8_t* __restrict__ out, int64_t out_stride) {
  __shared__ uint64_t x[312];
  __shared__ int wcnt[2][kMtThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint8_t* colors = out + blockIdx.x * out_stride;
  if (k == 1) {  // count_table.hpp:97: no draws
    for (int32_t v = t; v < n; v += blockDim.x) colors[v] = 0;
    return;
  }
  if (t == 0) {
    uint64_t s = seeds[blockIdx.x];
    x[0] = s;
    for (int j = 1; j < 312; ++j) { s = 6364136223846793005ULL * (s ^ (s >> 62)) + j; x[j] = s; }
  }
  __syncthreads();
  constexpr uint64_t U = 0xFFFFFFFF80000000ULL, L = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  const bool act = t < 156;
  int64_t base = 0;
  while (base < n) {
    uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0, o4 = 0;
    if (act) { o0 = x[t]; o1 = x[t + 1]; o2 = x[t + 156]; o3 = x[t + 156]; o4 = x[(t + 157) % 312]; }
    __syncthreads();
    uint64_t w0 = 0, w1 = 0;
    if (act) {
      uint64_t y = (o0 & U) | (o1 & L);
      w0 = o2 ^ (y >> 1) ^ ((y & 1) ? A : 0);        // word t (phase 1)
      x[t] = w0;
      if (t < 155) {
        y = (o3 & U) | (o4 & L);
        w1 = w0 ^ (y >> 1) ^ ((y & 1) ? A : 0);      // word 156+t reads new word t
        x[t + 156] = w1;
      }
    }
    __syncthreads();
    if (t == 155) {                                  // word 311: new x[0], new x[155]
      const uint64_t y = (o3 & U) | (x[0] & L);
      w1 = x[155] ^ (y >> 1) ^ ((y & 1) ? A : 0);
      x[311] = w1;
    }
    // temper
    auto temper = [](uint64_t z) {
      z ^= (z >> 29) & 0x5555555555555555ULL;
      z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
      z ^= (z << 37) & 0xFFF7EEE000000000ULL;
      return z ^ (z >> 43);
    };
    const uint64_t z0 = temper(w0), z1 = temper(w1);
    const bool r0 = act && z0 >= limit, r1 = act && z1 >= limit;
    if (!__syncthreads_or(r0 || r1)) {
      if (act) {
        const int64_t v0 = base + t, v1 = base + 156 + t;
        if (v0 < n) colors[v0] = static_cast<uint8_t>(z0 % static_cast<uint64_t>(k));
        if (v1 < n) colors[v1] = static_cast<uint8_t>(z1 % static_cast<uint64_t>(k));
      }
      base += 312;
    } else {
      // exclusive scan of rejection flags over word order 0..311
      const unsigned b0 = __ballot_sync(0xffffffffu, r0), b1 = __ballot_sync(0xffffffffu, r1);
      if (lane == 0) { wcnt[0][warp] = __popc(b0); wcnt[1][warp] = __popc(b1); }
      __syncthreads();
      int pre0 = 0, pre1 = 0, tot0 = 0, tot1 = 0;
      for (int w = 0; w < kMtThreads / 32; ++w) {
        if (w < warp) { pre0 += wcnt[0][w]; pre1 += wcnt[1][w]; }
        tot0 += wcnt[0][w];
        tot1 += wcnt[1][w];
      }
      const unsigned lt = (1u << lane) - 1u;
      pre0 += __popc(b0 & lt);
      pre1 += __popc(b1 & lt) + tot0;
      if (act) {
        const int64_t v0 = base + t - pre0, v1 = base + 156 + t - pre1;
        if (!r0 && v0 < n) colors[v0] = static_cast<uint8_t>(z0 % static_cast<uint64_t>(k));
        if (!r1 && v1 < n) colors[v1] = static_cast<uint8_t>(z1 % static_cast<uint64_t>(k));
      }
      base += 312 - tot0 - tot1;
      __syncthreads();
    }
  }
}

// ------------------------------------------------------- neighbour histogram
// P'[v, c] = |{u in N(v) : color(u) = c}| -- the SpMM of the adjacency with a
// one-hot leaf table, read from 1-byte colors instead of n x k floats.
// Warp per row; lane c accumulates color c via ballots.  Exact (integers).
__global__ void __launch_bounds__(256)
nbr_hist(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
         const uint8_t* __restrict__ colors, int32_t n, int k, float* __restrict__ H) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t pol = policy_evict_first();
  for (int64_t v = warp0; v < n; v += nw) {
    const int64_t b = row_ptr[v], e = row_ptr[v + 1];
    unsigned cnt = 0;
    for (int64_t j = b; j < e; j += 32) {
      const int c = j + lane < e ? colors[ld_stream_i32(col + j + lane, pol)] : 255;
      for (int cc = 0; cc < k; ++cc) {
        const unsigned m = __ballot_sync(0xffffffffu, c == cc);
        if (lane == cc) cnt += __popc(m);
      }
    }
    const int panels = (k + Z - 1) / Z;
    if (lane < panels * Z)
      H[static_cast<int64_t>(lane / Z) * n * Z + v * Z + (lane % Z)] =
          lane < k ? static_cast<float>(cnt) : 0.f;
  }
}

// ----------------------------------------------------------------- SpMM
// Y[:, panel] = A . X[:, panel] for every panel of the passive table.
// Work unit: a warp owns 8 segments (one per 4-lane group); segments are
// sorted by length (descending) on the host so the 8 groups of a warp run
// the same trip count, and the longest units are issued first.  Each group
// gathers one 64 B row panel per neighbour (4 x float4), accumulating in
// fp64 (SURVEY finding 3: hub rows up to 261K neighbours).  Blocks are
// panel-major, so all SMs sweep one panel at a time and it stays L2-resident.
constexpr int kSpmmWarps = 8;

__global__ void __launch_bounds__(kSpmmWarps * 32)
spmm_panels(const Seg* __restrict__ segs, int64_t ntasks, int64_t blocks_per_panel,
            const int32_t* __restrict__ col, const float* __restrict__ X,
            float* __restrict__ Y, double* __restrict__ partial, int32_t n, int npanels) {
  const int lane = threadIdx.x & 31, g = lane >> 2, l = lane & 3;
  const int64_t panel = blockIdx.x / blocks_per_panel;
  const int64_t task = (blockIdx.x % blocks_per_panel) * kSpmmWarps + (threadIdx.x >> 5);
  if (task >= ntasks) return;
  const Seg s = segs[task * 8 + g];
  const int maxlen = __shfl_sync(0xffffffffu, s.len, 0);  // sorted: group 0 is longest
  const float* Xp = X + panel * static_cast<int64_t>(n) * Z + l * 4;
  const int32_t* cp = col + s.e_begin;
  const uint64_t pstream = policy_evict_first(), pkeep = policy_evict_last();
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int t = 0; t < maxlen; t += 8) {
    const int i0 = t + l < s.len ? ld_stream_i32(cp + t + l, pstream) : -1;
    const int i1 = t + 4 + l < s.len ? ld_stream_i32(cp + t + 4 + l, pstream) : -1;
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int u = __shfl_sync(0xffffffffu, j < 4 ? i0 : i1, (g << 2) | (j & 3));
      v[j] = u >= 0 ? ld_keep_f4(Xp + static_cast<int64_t>(u) * Z, pkeep) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) { a0 += v[j].x; a1 += v[j].y; a2 += v[j].z; a3 += v[j].w; }
  }
  if (s.dst >= 0) {
    if (s.dst != kSkip)
      st_stream_f4(Y + panel * static_cast<int64_t>(n) * Z + static_cast<int64_t>(s.dst) * Z + l * 4,
                   make_float4(static_cast<float>(a0), static_cast<float>(a1),
                               static_cast<float>(a2), static_cast<float>(a3)), pstream);
  } else {
    double* pp = partial + ((static_cast<int64_t>(-1 - s.dst) * npanels + panel) * Z + l * 4);
    reinterpret_cast<double2*>(pp)[0] = make_double2(a0, a1);
    reinterpret_cast<double2*>(pp)[1] = make_double2(a2, a3);
  }
}

// Sum the fp64 partials of split rows in segment order (deterministic).
__global__ void spmm_fixup(const int32_t* __restrict__ rows, const int32_t* __restrict__ slot_begin,
                           int nrows, const double* __restrict__ partial, float* __restrict__ Y,
                           int32_t n, int npanels) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t total = static_cast<int64_t>(nrows) * npanels * Z;
  if (i >= total) return;
  const int z = i % Z;
  const int64_t rp = i / Z;
  const int panel = rp % npanels;
  const int r = static_cast<int>(rp / npanels);
  double acc = 0;
  for (int s = slot_begin[r]; s < slot_begin[r + 1]; ++s)
    acc += partial[(static_cast<int64_t>(s) * npanels + panel) * Z + z];
  Y[static_cast<int64_t>(panel) * n * Z + static_cast<int64_t>(rows[r]) * Z + z] = static_cast<float>(acc);
}

// ------------------------------------------------------------------- eMA
// M_s[v,S] = sum_p M_a[v, A(S,p)] * P'[v, P(S,p)]  over the by-parent split
// pairs (color_index.hpp:97-98,131-165).  A CTA owns 32 consecutive
// vertices; both input rows are staged into smem column-major with a
// 33-float pitch (lane = vertex -> conflict-free reads).  Warp w computes
// whole output panels (16 parent columns) in registers and writes each
// 32 x 16 block (2 KB, contiguous in the panel layout) through an smem
// transpose with float4 stores.  ALEAF: the active child is a leaf, so
// M_a[v, A] = [A == color(v)] and nothing is staged for it.  ROOT: one
// parent column, fp64 output + per-tile fp64 partial of the total; the
// warps split the pair list and reduce in a fixed order.
template <typename AccT, bool ALEAF, bool ROOT, bool STAGED>
__global__ void __launch_bounds__(kEmaWarps * 32)
ema_tile(const float* __restrict__ Am, const float* __restrict__ Pm,
         const uint8_t* __restrict__ colors, const int2* __restrict__ split, int pairs,
         int Ca, int Cp, int Cs, int32_t n, float* __restrict__ out,
         double* __restrict__ root_out, double* __restrict__ root_acc,
         double* __restrict__ tile_tot) {
  extern __shared__ float smem[];
  constexpr int P = kTileV + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t v0 = static_cast<int64_t>(blockIdx.x) * kTileV;
  const int64_t v = v0 + lane;
  const bool valid = v < n;
  float* sA = smem;                                   // [Ca][33] (unless ALEAF)
  float* sP = smem + (ALEAF || !STAGED ? 0 : Ca * P); // [Cp][33]
  float* sO = sP + (STAGED ? Cp * P : 0) + warp * (kTileV * (Z + 1));  // per-warp transpose
  const int my_color = valid ? colors[v] : -1;

  if (STAGED) {
    auto stage = [&](const float* T, int C, float* dst) {
      const int panels = (C + Z - 1) / Z;
      for (int i = tid; i < panels * kTileV * (Z / 4); i += blockDim.x) {
        const int p = i / (kTileV * (Z / 4)), r = i % (kTileV * (Z / 4));
        const int vv = r / (Z / 4), z4 = (r % (Z / 4)) * 4;
        float4 x = make_float4(0, 0, 0, 0);
        if (v0 + vv < n) x = *reinterpret_cast<const float4*>(T + (static_cast<int64_t>(p) * n + v0 + vv) * Z + z4);
        const int c = p * Z + z4;
        if (c + 0 < C) dst[(c + 0) * P + vv] = x.x;
        if (c + 1 < C) dst[(c + 1) * P + vv] = x.y;
        if (c + 2 < C) dst[(c + 2) * P + vv] = x.z;
        if (c + 3 < C) dst[(c + 3) * P + vv] = x.w;
      }
    };
    if (!ALEAF) stage(Am, Ca, sA);
    stage(Pm, Cp, sP);
    __syncthreads();
  }
  auto aval = [&](int ia) -> float {
    if (ALEAF) return ia == my_color ? 1.f : 0.f;
    if (STAGED) return sA[ia * P + lane];
    return valid ? Am[(static_cast<int64_t>(ia / Z) * n + v) * Z + ia % Z] : 0.f;
  };
  auto pval = [&](int ip) -> float {
    if (STAGED) return sP[ip * P + lane];
    return valid ? Pm[(static_cast<int64_t>(ip / Z) * n + v) * Z + ip % Z] : 0.f;
  };

  if (ROOT) {
    __shared__ double red[kEmaWarps][kTileV];
    AccT acc = 0;
    for (int p = warp; p < pairs; p += kEmaWarps) {
      const int2 s = split[p];
      acc += static_cast<AccT>(aval(s.x)) * static_cast<AccT>(pval(s.y));
    }
    red[warp][lane] = static_cast<double>(acc);
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
      // fixed-order tile total
      for (int o = 16; o; o >>= 1) tot += __shfl_down_sync(0xffffffffu, tot, o);
      if (lane == 0) tile_tot[blockIdx.x] = tot;
    }
    return;
  }

  const int opanels = (Cs + Z - 1) / Z;
  for (int po = warp; po < opanels; po += kEmaWarps) {
    float r[Z];
#pragma unroll
    for (int z = 0; z < Z; ++z) {
      const int S = po * Z + z;
      AccT acc = 0;
      if (S < Cs) {
        const int2* sp = split + static_cast<int64_t>(S) * pairs;
        for (int p = 0; p < pairs; ++p) {
          const int2 s = sp[p];
          acc += static_cast<AccT>(aval(s.x)) * static_cast<AccT>(pval(s.y));
        }
      }
      r[z] = static_cast<float>(acc);
    }
    // transpose 32 vertices x 16 columns through smem, then 2 KB of float4
#pragma unroll
    for (int z = 0; z < Z; ++z) sO[lane * (Z + 1) + z] = r[z];
    __syncwarp();
    float* dst = out + (static_cast<int64_t>(po) * n + v0) * Z;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = q * 32 + lane;           // float4 index within the 32x16 block
      const int vv = idx >> 2, z4 = (idx & 3) * 4;
      if (v0 + vv < n) {
        const float* s = sO + vv * (Z + 1) + z4;
        *reinterpret_cast<float4*>(dst + vv * Z + z4) = make_float4(s[0], s[1], s[2], s[3]);
      }
    }
    __syncwarp();
  }
}

// Deterministic fp64 sum of the per-tile totals (engines.hpp:125-129; the
// reference's sequential sum differs only at the 1e-16 level).
__global__ void root_reduce(const double* __restrict__ tile_tot, int64_t ntiles,
                            double* __restrict__ total) {
  __shared__ double red[1024];
  double s = 0;
  for (int64_t i = threadIdx.x; i < ntiles; i += blockDim.x) s += tile_tot[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = red[0];
}

}  // namespace dev
}  // namespace tcg
