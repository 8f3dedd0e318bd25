// kernels_rt.cuh -- eMA over ROOTED tables (same-color vertex tiles).
//
// Every non-root table M_x[v,S] is zero unless S contains color(v) (the root
// of T_x sits on v).  With v's color c fixed, the eMA of a node (s, a, p) is
// the eMA of the (k-1)-color problem (s-1, a-1, p): output S' = S minus c,
// active Sa' = Sa minus c, passive Sp (which never contains c), all indexed
// by the combinadic of the colors relabeled to [0, k-1) ("relabeled index").
// Vertices are sorted by color once per coloring (vsort_*), so a 32-vertex
// tile shares c and every lane runs the same split pairs:
//   * the active table is stored ROOTED (RR): column j = relabeled index of
//     S minus c (C(k-1, s-1) columns) -- staged as is;
//   * P' (full, or group-major from the rooted SpMM) is staged through a
//     per-color map: storage column -> relabeled index, or -1 when it
//     contains c (those values are never used);
//   * the output is RR, or -- for a passive child feeding the rooted SpMM --
//     the SpMM's slot layout (RS) through a per-color output map.
// FMAs drop to a/k of the full-table eMA, table bytes to s/k.
#pragma once

namespace tcg {
namespace dev {

// ----------------------------------------------- per-coloring vertex sort
constexpr int kVsChunk = 4096;  // vertices per CTA

__global__ void __launch_bounds__(256)
vsort_count(const uint8_t* __restrict__ colors, int32_t n, int k, int* __restrict__ cnt) {
  __shared__ int h[32];
  if (threadIdx.x < 32) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t b = static_cast<int64_t>(blockIdx.x) * kVsChunk;
  for (int i = threadIdx.x; i < kVsChunk; i += blockDim.x) {
    const int64_t v = b + i;
    if (v < n) atomicAdd(&h[colors[v]], 1);
  }
  __syncthreads();
  if (threadIdx.x < k) cnt[blockIdx.x * k + threadIdx.x] = h[threadIdx.x];
}

// One CTA: per-(chunk, color) offsets (color-major, chunk order) in place,
// and the tile table: tile t = {color, first sorted position, count}, tiles
// numbered color by color; unused entries get color -1.
__global__ void __launch_bounds__(1024)
vsort_scan(int* __restrict__ cnt, int nchunks, int k, int4* __restrict__ tiles, int max_tiles) {
  // warp c scans color c's chunk counts (chunk order); then the tile table
  __shared__ int tot[32], start[33], tstart[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < k) {
    int run = 0;
    for (int b0 = 0; b0 < nchunks; b0 += 32) {
      const int b = b0 + lane;
      const int x = b < nchunks ? cnt[b * k + warp] : 0;
      int incl = x;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (b < nchunks) cnt[b * k + warp] = run + incl - x;  // color-local offset
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) tot[warp] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    start[0] = tstart[0] = 0;
    for (int q = 0; q < k; ++q) {
      start[q + 1] = start[q] + tot[q];
      tstart[q + 1] = tstart[q] + (tot[q] + 31) / 32;
    }
  }
  __syncthreads();
  if (warp < k)
    for (int b = lane; b < nchunks; b += 32) cnt[b * k + warp] += start[warp];
  for (int t = threadIdx.x; t < max_tiles; t += blockDim.x) {
    int cc = -1;
    for (int q = 0; q < k; ++q)
      if (t >= tstart[q] && t < tstart[q + 1]) cc = q;
    if (cc < 0) {
      tiles[t] = make_int4(-1, 0, 0, 0);
    } else {
      const int s0 = start[cc] + 32 * (t - tstart[cc]);
      tiles[t] = make_int4(cc, s0, min(32, start[cc + 1] - s0), 0);
    }
  }
}

// Stable scatter: warp w of a chunk owns 512 consecutive vertices.
__global__ void __launch_bounds__(256)
vsort_scatter(const uint8_t* __restrict__ colors, int32_t n, int k, const int* __restrict__ off,
              int32_t* __restrict__ sorted) {
  __shared__ int wc[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * kVsChunk + warp * (kVsChunk / 8);
  wc[warp][lane] = 0;
  __syncwarp();
  for (int i = 0; i < kVsChunk / 8; i += 32) {
    const int64_t v = b + i + lane;
    const int c = v < n ? colors[v] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, c);
    if (c >= 0 && (same & lt) == 0) wc[warp][c] += __popc(same);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < k) {  // warp-major prefix per color, plus the chunk offset
    int run = off[blockIdx.x * k + threadIdx.x];
    for (int w = 0; w < 8; ++w) {
      const int x = wc[w][threadIdx.x];
      wc[w][threadIdx.x] = run;
      run += x;
    }
  }
  __syncthreads();
  for (int i = 0; i < kVsChunk / 8; i += 32) {
    const int64_t v = b + i + lane;
    const int c = v < n ? colors[v] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, c);
    const int pos = c >= 0 ? wc[warp][c] + __popc(same & lt) : 0;
    __syncwarp();
    if (c >= 0) {
      sorted[pos] = static_cast<int32_t>(v);
      if ((same & lt) == 0) wc[warp][c] += __popc(same);
    }
    __syncwarp();
  }
}

// Stage the rows of the (up to 32) tile vertices of a panel table with C
// storage columns into smem [row][kSpitch] (lane = vertex).  map (nullable):
// storage column -> smem row, or -1 to drop.  Missing vertices stage zeros.
template <int kStageU>
__device__ __forceinline__ void stage_rows(const float* __restrict__ T, int C, int32_t n,
                                           const int32_t* __restrict__ vids, float* dst,
                                           const int32_t* __restrict__ map, int tid = threadIdx.x,
                                           int nth = blockDim.x) {
  const int panels = num_panels(C);
  const int zl = last_panel_width(C);
  const int full4 = (panels - 1) * kTileV * (kZ / 4);
  const int total4 = full4 + kTileV * (zl / 4);
  const int lq_last = zl == 32 ? 3 : (zl == 16 ? 2 : 1);  // log2(float4s per row) of the last panel
  for (int base = tid; base < total4; base += nth * kStageU) {
    float4 x[kStageU];
    int c0[kStageU], vv[kStageU];
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int f = base + u * nth;
      int p, r, lq;
      if (f < full4) { p = f >> 8; r = f & 255; lq = 3; }  // kTileV * 8 float4s per full panel tile
      else { p = panels - 1; r = f - full4; lq = lq_last; }
      vv[u] = r >> lq;
      const int q = r & ((1 << lq) - 1);
      c0[u] = p * kZ + q * 4;
      x[u] = make_float4(0, 0, 0, 0);
      const int v = f < total4 ? vids[vv[u]] : -1;
      if (v >= 0 && c0[u] < C)
        x[u] = __ldg(reinterpret_cast<const float4*>(T + static_cast<int64_t>(p) * n * kZ + (static_cast<int64_t>(v) << (lq + 2)) + q * 4));
      if (f >= total4) c0[u] = C;
    }
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int c = c0[u];
      if (c >= C) continue;
      if (map) {
        const int4 m = make_int4(__ldg(map + c), c + 1 < C ? __ldg(map + c + 1) : -1,
                                 c + 2 < C ? __ldg(map + c + 2) : -1, c + 3 < C ? __ldg(map + c + 3) : -1);
        if (m.x >= 0) dst[m.x * kSpitch + vv[u]] = x[u].x;
        if (m.y >= 0) dst[m.y * kSpitch + vv[u]] = x[u].y;
        if (m.z >= 0) dst[m.z * kSpitch + vv[u]] = x[u].z;
        if (m.w >= 0) dst[m.w * kSpitch + vv[u]] = x[u].w;
      } else {
        dst[(c + 0) * kSpitch + vv[u]] = x[u].x;
        if (c + 1 < C) dst[(c + 1) * kSpitch + vv[u]] = x[u].y;
        if (c + 2 < C) dst[(c + 2) * kSpitch + vv[u]] = x[u].z;
        if (c + 3 < C) dst[(c + 3) * kSpitch + vv[u]] = x[u].w;
      }
    }
  }
}

// Output of 8 consecutive relabeled columns [c0, c0+8) of vertex v: RR (omap
// null: the table has Ws columns, written as two float4) or RS (column ->
// slot through omap, table of Cout columns).
__device__ __forceinline__ void rt_write8(float* __restrict__ out, int Ws, int Cout, const int32_t* __restrict__ omap,
                                          int32_t n, int64_t v, int c0, const float (&r)[8]) {
  if (!omap) {
    const int zw = panel_width(Ws, c0 / kZ);
    float* dst = out + static_cast<int64_t>(c0 / kZ) * n * kZ + v * zw + (c0 % kZ);
    if (c0 + 4 <= Ws || (c0 % kZ) + 4 <= zw) reinterpret_cast<float4*>(dst)[0] = make_float4(r[0], r[1], r[2], r[3]);
    if ((c0 % kZ) + 8 <= zw) reinterpret_cast<float4*>(dst)[1] = make_float4(r[4], r[5], r[6], r[7]);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (c0 + j < Ws) out[panel_offset(Cout, n, v, __ldg(omap + c0 + j))] = r[j];
  }
}

// Generic node (and the active-leaf copy) on a same-color tile.  Warp w
// computes chunks of 8 output columns for the tile's 32 vertices.
template <bool ALEAF>
__global__ void __launch_bounds__(kEmaWarps * 32)
ema_rt_node(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca, const float* __restrict__ Pm, int Cpt,
            const int32_t* __restrict__ pmap, int Wp, const int32_t* __restrict__ vsorted,
            const int4* __restrict__ tiles, const uint32_t* __restrict__ packed, int pairs, int Ws,
            const int32_t* __restrict__ omap, const int32_t* __restrict__ imap, int Cout, int32_t n,
            float* __restrict__ out) {
  extern __shared__ float smem[];
  __shared__ int32_t vids[32];
  const int4 tile = tiles[blockIdx.x];
  if (tile.x < 0) return;
  const int c = tile.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 32) vids[threadIdx.x] = static_cast<int>(threadIdx.x) < tile.z ? vsorted[tile.y + threadIdx.x] : -1;
  __syncthreads();
  float* sA = smem;
  float* sP = smem + (ALEAF ? 0 : Wa * kSpitch);
  if (!ALEAF) stage_rows<1>(Am, Ca, n, vids, sA, amap ? amap + static_cast<int64_t>(c) * Ca : nullptr);
  stage_rows<1>(Pm, Cpt, n, vids, sP, pmap + static_cast<int64_t>(c) * Cpt);
  __syncthreads();
  const int64_t v = vids[lane];
  const int32_t* om = omap ? omap + static_cast<int64_t>(c) * Ws : nullptr;
  // RS output: staged in smem [Ws][kSpitch], then written as coalesced slot
  // rows through the per-color inverse map (imap: slot -> output column)
  float* sO = smem + (ALEAF ? 0 : Wa * kSpitch) + Wp * kSpitch;
  const int nchunks = (Ws + 7) / 8;
  for (int q = warp; q < nchunks; q += blockDim.x >> 5) {
    float r[8];
    if (ALEAF) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = q * 8 + j < Ws ? sP[(q * 8 + j) * kSpitch + lane] : 0.f;
    } else {
      const int nv = min(8, Ws - q * 8);
      const uint32_t* sp = packed + static_cast<int64_t>(q) * 8 * pairs;
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = 0.f;
      for (int pb = 0; pb < pairs; pb += 32) {
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = (j < nv && pb + lane < pairs) ? __ldg(sp + j * pairs + pb + lane) : 0u;
        const int cnt = min(32, pairs - pb);
        for (int pp = 0; pp < cnt; ++pp) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t s = __shfl_sync(0xffffffffu, w[j], pp);
            r[j] = fmaf(sA[(s & 0xFFFFu) * kSpitch + lane], sP[(s >> 16) * kSpitch + lane], r[j]);
          }
        }
      }
    }
    if (om && imap) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (q * 8 + j < Ws) sO[(q * 8 + j) * kSpitch + lane] = r[j];
    } else if (v >= 0) {
      rt_write8(out, Ws, Cout, om, n, v, q * 8, r);
    }
  }
  if (om && imap) {
    __syncthreads();
    const int32_t* im = imap + static_cast<int64_t>(c) * Cout;
    const int pout = num_panels(Cout), zout = last_panel_width(Cout);
    for (int rr = warp; rr < 32; rr += blockDim.x >> 5) {
      const int64_t u = vids[rr];
      if (u < 0) continue;
      for (int p = 0; p < pout; ++p) {
        const int zp = p == pout - 1 ? zout : kZ;
        if (lane < zp) {
          const int j = p * kZ + lane < Cout ? __ldg(im + p * kZ + lane) : -1;
          out[static_cast<int64_t>(p) * n * kZ + u * zp + lane] = j >= 0 ? sO[j * kSpitch + rr] : 0.f;
        }
      }
    }
  }
}

// 16-byte global -> shared copy that bypasses registers (LDGSTS); wait with cp_async_wait_all_()
__device__ __forceinline__ void cp_async16_(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all_() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Active-leaf node: M_s[v,S] = P'[v, S minus c] -- a per-color column
// permutation of the vertex's P' row: out[v, i] = P'[v, cmap[c][i]] (0 where
// -1).  A CTA stages the full P' rows of `vpb` consecutive vertices in smem
// (coalesced 128 B panel rows), then writes the output rows panel by panel
// (coalesced as well).  Natural vertex order, no tiles.
__global__ void __launch_bounds__(256)
ema_rt_copy(const float* __restrict__ Pm, int Cpt, const uint8_t* __restrict__ colors,
            const int32_t* __restrict__ cmap, int Cout, int32_t n, int vpb, int L, float* __restrict__ out) {
  // L lanes per vertex row (a power of two <= 32, sized to the rows on the host)
  extern __shared__ float crow[];
  const int lane = threadIdx.x & 31, sub = lane & (L - 1);
  const int grp = static_cast<int>(threadIdx.x) / L, ngrp = blockDim.x / L;
  const int pin = num_panels(Cpt), zin = last_panel_width(Cpt);
  const int rf = (pin - 1) * kZ + zin;  // floats of one panel-padded row
  const int64_t u0 = static_cast<int64_t>(blockIdx.x) * vpb;
  if (L == 32) {
    // wide rows (one warp per row would leave warps idle whenever vpb is not a multiple of the
    // warp count): every warp works on every row -- the whole CTA stages a row's float4s, and
    // warp w writes output panels w, w + 8, ...
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = 0; r < vpb && u0 + r < n; ++r) {
      const int64_t u = u0 + r;
      for (int c4 = threadIdx.x * 4; c4 < rf; c4 += blockDim.x * 4) {
        const int p = c4 >> 5, z = c4 & 31;
        const int zp = p == pin - 1 ? zin : kZ;
        cp_async16_(crow + r * rf + c4, Pm + static_cast<int64_t>(p) * n * kZ + u * zp + z);
      }
    }
    cp_async_wait_all_();
    __syncthreads();
    const int pout = num_panels(Cout), zout = last_panel_width(Cout);
    for (int r = 0; r < vpb && u0 + r < n; ++r) {
      const int64_t u = u0 + r;
      const int32_t* cm = cmap + static_cast<int64_t>(colors[u]) * Cout;
      for (int p = warp; p < pout; p += nw) {
        const int zp = p == pout - 1 ? zout : kZ;
        if (lane < zp) {
          const int col = p * kZ + lane;
          const int src = col < Cout ? __ldg(cm + col) : -1;
          out[static_cast<int64_t>(p) * n * kZ + u * zp + lane] = src >= 0 ? crow[r * rf + src] : 0.f;
        }
      }
    }
    return;
  }
  for (int r = grp; r < vpb; r += ngrp) {  // stage: 128 B panel rows, float4 per lane
    const int64_t u = u0 + r;
    if (u >= n) break;
    for (int c4 = sub * 4; c4 < rf; c4 += L * 4) {
      const int p = c4 >> 5, z = c4 & 31;
      const int zp = p == pin - 1 ? zin : kZ;
      cp_async16_(crow + r * rf + c4, Pm + static_cast<int64_t>(p) * n * kZ + u * zp + z);
    }
  }
  cp_async_wait_all_();
  __syncthreads();
  const int pout = num_panels(Cout), zout = last_panel_width(Cout);
  for (int r = grp; r < vpb; r += ngrp) {  // write: consecutive lanes -> consecutive slots of a row
    const int64_t u = u0 + r;
    if (u >= n) break;
    const int32_t* cm = cmap + static_cast<int64_t>(colors[u]) * Cout;
    for (int p = 0; p < pout; ++p) {
      const int zp = p == pout - 1 ? zout : kZ;
      for (int t = sub; t < zp; t += L) {
        const int col = p * kZ + t;
        const int src = col < Cout ? __ldg(cm + col) : -1;
        out[static_cast<int64_t>(p) * n * kZ + u * zp + t] = src >= 0 ? crow[r * rf + src] : 0.f;
      }
    }
  }
}

// ema_rt_node with one WARP per tile (narrow nodes): every warp stages its
// own tile's rows into its smem slice and computes all of the tile's output
// chunks, so 8 tiles per CTA (and 2-4 CTAs per SM) are in flight instead of
// one -- the narrow nodes are latency-bound on the staging round trips.
// Slice layout: A [Wa][kSpitch], P [Wp][kSpitch], RS output tile [Ws][kSpitch].
__global__ void __launch_bounds__(256)
ema_rt_node_w(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca, const float* __restrict__ Pm,
              int Cpt, const int32_t* __restrict__ pmap, int Wp, const int32_t* __restrict__ vsorted,
              const int4* __restrict__ tiles, int ntiles, const uint32_t* __restrict__ packed, int pairs, int Ws,
              const int32_t* __restrict__ omap, const int32_t* __restrict__ imap, int Cout, int32_t n, int slice,
              float* __restrict__ out) {
  extern __shared__ float smem[];
  __shared__ int32_t vids_all[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * (blockDim.x >> 5) + warp;
  if (t >= ntiles) return;
  const int4 tile = tiles[t];
  if (tile.x < 0) return;
  const int c = tile.x;
  int32_t* vids = vids_all[warp];
  vids[lane] = lane < tile.z ? vsorted[tile.y + lane] : -1;
  __syncwarp();
  float* sA = smem + static_cast<int64_t>(warp) * slice;
  float* sP = sA + Wa * kSpitch;
  float* sO = sP + Wp * kSpitch;
  stage_rows<4>(Am, Ca, n, vids, sA, amap ? amap + static_cast<int64_t>(c) * Ca : nullptr, lane, 32);
  stage_rows<4>(Pm, Cpt, n, vids, sP, pmap + static_cast<int64_t>(c) * Cpt, lane, 32);
  __syncwarp();
  const int64_t v = vids[lane];
  const int32_t* om = omap ? omap + static_cast<int64_t>(c) * Ws : nullptr;
  const int nchunks = (Ws + 7) / 8;
  for (int q = 0; q < nchunks; ++q) {
    float r[8];
    const int nv = min(8, Ws - q * 8);
    const uint32_t* sp = packed + static_cast<int64_t>(q) * 8 * pairs;
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = 0.f;
    for (int pb = 0; pb < pairs; pb += 32) {
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = (j < nv && pb + lane < pairs) ? __ldg(sp + j * pairs + pb + lane) : 0u;
      const int cnt = min(32, pairs - pb);
      for (int pp = 0; pp < cnt; ++pp) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t s = __shfl_sync(0xffffffffu, w[j], pp);
          r[j] = fmaf(sA[(s & 0xFFFFu) * kSpitch + lane], sP[(s >> 16) * kSpitch + lane], r[j]);
        }
      }
    }
    if (om && imap) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (q * 8 + j < Ws) sO[(q * 8 + j) * kSpitch + lane] = r[j];
    } else if (v >= 0) {
      rt_write8(out, Ws, Cout, om, n, v, q * 8, r);
    }
  }
  if (om && imap) {
    __syncwarp();
    const int32_t* im = imap + static_cast<int64_t>(c) * Cout;
    const int pout = num_panels(Cout), zout = last_panel_width(Cout);
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t u = vids[rr];
      if (u < 0) continue;
      for (int p = 0; p < pout; ++p) {
        const int zp = p == pout - 1 ? zout : kZ;
        if (lane < zp) {
          const int j = p * kZ + lane < Cout ? __ldg(im + p * kZ + lane) : -1;
          out[static_cast<int64_t>(p) * n * kZ + u * zp + lane] = j >= 0 ? sO[j * kSpitch + rr] : 0.f;
        }
      }
    }
  }
}

// Wide nodes over a LEAF passive child (p = 1) whose 32-vertex tile does not
// fit (cfg4's (7,6,1)): out'[S'] = sum over d in S' of A'[S' minus d] *
// H[v, d] (relabeled past c(v)) -- s' terms per output, so the register-blocked
// micro-patterns of ema_rtv_blocked are all overhead here.  A CTA stages the A
// rows and histograms of kPleafV vertices; a thread takes output columns and,
// per drop-table entry {A index | d << 16} (s' per output, read once),
// accumulates all kPleafV vertices into the vertices' output rows staged in
// smem (storage order: RR columns, or the RS slots of the parent's SpMM),
// which warps then write as whole 128 B panel rows.
template <int kPleafV, int SP>  // SP: compile-time s' of the packed drop rows (1..6), 0 = unpacked rows
__global__ void __launch_bounds__(256)
ema_rtv_pleaf(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca,
              const float* __restrict__ Pm, int Cpt, const int32_t* __restrict__ pmap,
              const uint8_t* __restrict__ colors, const uint32_t* __restrict__ drop, int sp, int Ws,
              const int32_t* __restrict__ omap, int Cout, int32_t n, int slice, int oslice, float* __restrict__ out) {
  extern __shared__ float smem[];
  __shared__ int cvs[kPleafV];
  float* sO = smem + kPleafV * slice;  // [kPleafV][oslice]: output rows in storage order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int pa = num_panels(Ca), za = last_panel_width(Ca);
  const int tot4 = ((pa - 1) * kZ + za) / 4;
  for (int64_t v0 = static_cast<int64_t>(blockIdx.x) * kPleafV; v0 < n; v0 += static_cast<int64_t>(gridDim.x) * kPleafV) {
    __syncthreads();
    if (threadIdx.x < kPleafV) cvs[threadIdx.x] = v0 + threadIdx.x < n ? colors[v0 + threadIdx.x] : 0;
    // the whole CTA stages the kPleafV A rows (through amap when the table is
    // packed or virtual) -- every thread's loads are in flight at once -- and
    // one warp per vertex its relabeled histogram
    for (int idx = threadIdx.x; idx < kPleafV * tot4; idx += blockDim.x) {
      const int vv = idx / tot4, f = idx - vv * tot4;
      const int64_t v = v0 + vv;
      float* sA = smem + static_cast<int64_t>(vv) * slice;
      const int c0 = f * 4, p = c0 / kZ, z4 = c0 % kZ;
      if (v >= n) {
        if (c0 < Wa) sA[c0] = 0.f;
        if (c0 + 1 < Wa) sA[c0 + 1] = 0.f;
        if (c0 + 2 < Wa) sA[c0 + 2] = 0.f;
        if (c0 + 3 < Wa) sA[c0 + 3] = 0.f;
        continue;
      }
      const int zw = p == pa - 1 ? za : kZ;
      const float4 x = __ldg(reinterpret_cast<const float4*>(Am + static_cast<int64_t>(p) * n * kZ + v * zw + z4));
      if (!amap) {
        if (c0 < Wa) sA[c0] = x.x;
        if (c0 + 1 < Wa) sA[c0 + 1] = x.y;
        if (c0 + 2 < Wa) sA[c0 + 2] = x.z;
        if (c0 + 3 < Wa) sA[c0 + 3] = x.w;
      } else {
        const int32_t* am = amap + static_cast<int64_t>(colors[v]) * Ca;
        const int m0 = c0 < Ca ? __ldg(am + c0) : -1, m1 = c0 + 1 < Ca ? __ldg(am + c0 + 1) : -1;
        const int m2 = c0 + 2 < Ca ? __ldg(am + c0 + 2) : -1, m3 = c0 + 3 < Ca ? __ldg(am + c0 + 3) : -1;
        if (m0 >= 0) sA[m0] = x.x;
        if (m1 >= 0) sA[m1] = x.y;
        if (m2 >= 0) sA[m2] = x.z;
        if (m3 >= 0) sA[m3] = x.w;
      }
    }
    for (int vv = warp; vv < kPleafV; vv += nw) {
      const int64_t v = v0 + vv;
      float* sH = smem + static_cast<int64_t>(vv) * slice + slice - 32;
      if (v >= n) {
        sH[lane] = 0.f;
        continue;
      }
      const int c = colors[v];
      if (lane < Cpt) {  // pmap: storage column -> d' (or -1 for c(v))
        const int d = __ldg(pmap + static_cast<int64_t>(c) * Cpt + lane);
        if (d >= 0) sH[d] = __ldg(Pm + v * panel_width(Cpt, 0) + lane);
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < Ws; j += blockDim.x) {
      float acc[kPleafV];
#pragma unroll
      for (int vv = 0; vv < kPleafV; ++vv) acc[vv] = 0.f;
      if constexpr (SP > 0) {  // (s' <= 6, k - 1 <= 16) six 16-bit A indices + six 4-bit colours in one 16 B load
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(drop) + j);
        const uint32_t w[3] = {q.x, q.y, q.z};
        const float* sHh = smem + slice - 32;
#pragma unroll
        for (int i = 0; i < SP; ++i) {
          const int ia = static_cast<int>((w[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu);
          const int ih = static_cast<int>((q.w >> (4 * i)) & 0xFu);
#pragma unroll
          for (int vv = 0; vv < kPleafV; ++vv) acc[vv] = fmaf(smem[vv * slice + ia], sHh[vv * slice + ih], acc[vv]);
        }
      } else {
        const uint32_t* dr = drop + static_cast<int64_t>(j) * sp;
        for (int i = 0; i < sp; ++i) {
          const uint32_t e = __ldg(dr + i);
          const int ia = static_cast<int>(e & 0xFFFFu), ih = static_cast<int>(e >> 16) + slice - 32;
#pragma unroll
          for (int vv = 0; vv < kPleafV; ++vv) acc[vv] = fmaf(smem[vv * slice + ia], smem[vv * slice + ih], acc[vv]);
        }
      }
#pragma unroll
      for (int vv = 0; vv < kPleafV; ++vv) {
        const int32_t* om = omap ? omap + static_cast<int64_t>(cvs[vv]) * Ws : nullptr;
        const int slot = om ? __ldg(om + j) : j;
        if (slot >= 0) sO[vv * oslice + slot] = acc[vv];
      }
    }
    __syncthreads();
    // whole panel rows: warp w writes (vertex, panel) rows w, w + nw, ...
    const int Cst = omap ? Cout : Ws;
    const int po = num_panels(Cst), zo = last_panel_width(Cst);
#pragma unroll
    for (int vv = 0; vv < kPleafV; ++vv) {
      const int64_t v = v0 + vv;
      if (v >= n) break;
      for (int p = warp; p < po; p += nw) {
        const int zp = p == po - 1 ? zo : kZ;
        if (lane < zp) {
          const int col = p * kZ + lane;
          out[static_cast<int64_t>(p) * n * kZ + v * zp + lane] = col < Cst ? sO[vv * oslice + col] : 0.f;
        }
      }
    }
  }
}

// Register-blocked eMA (see ema_blocked) on a same-color tile of the (k-1)
// problem; descriptors from build_blocked(k-1, s-1, a-1).
// blocks of a group are sorted by pattern; BlockDesc.pad of a run's first
// block holds the run length, so the pattern dispatch happens once per run
#define TCG_IJR(I, J)                                                                       \
  case I * 8 + J:                                                                           \
    for (int q = 0; q < len; ++q) {                                                         \
      const BlockDesc bd = q == 0 ? h : blocks[b + q];                                      \
      micro_block<I, J>(sA + bd.a_off * kSpitch + lane, sP + bd.p_off * kSpitch + lane, acc); \
    }                                                                                       \
    break;

constexpr int kRtBlockedThreads = 512;  // 2 CTAs x 16 warps per SM (64 registers, 2 x 87 KB smem at k=12)
__global__ void __launch_bounds__(kRtBlockedThreads, 2)
ema_rt_blocked(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca, const float* __restrict__ Pm, int Cpt,
               const int32_t* __restrict__ pmap, int Wp, const int32_t* __restrict__ vsorted,
               const int4* __restrict__ tiles, const GroupDesc* __restrict__ groups, int ngroups,
               const BlockDesc* __restrict__ blocks, int Ws, const int32_t* __restrict__ omap, int Cout,
               int32_t n, float* __restrict__ out) {
  extern __shared__ float smem[];
  __shared__ int next_group;
  __shared__ int32_t vids[32];
  const int4 tile = tiles[blockIdx.x];
  if (tile.x < 0) return;
  const int c = tile.x;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) vids[threadIdx.x] = static_cast<int>(threadIdx.x) < tile.z ? vsorted[tile.y + threadIdx.x] : -1;
  if (threadIdx.x == 0) next_group = blockDim.x / 32;
  __syncthreads();
  float* sA = smem;
  float* sP = smem + Wa * kSpitch;
  stage_rows<8>(Am, Ca, n, vids, sA, amap ? amap + static_cast<int64_t>(c) * Ca : nullptr);
  stage_rows<8>(Pm, Cpt, n, vids, sP, pmap + static_cast<int64_t>(c) * Cpt);
  __syncthreads();
  const int64_t v = vids[lane];
  const int32_t* om = omap ? omap + static_cast<int64_t>(c) * Ws : nullptr;
  for (int gi = threadIdx.x >> 5; gi < ngroups;) {
    const GroupDesc gd = groups[gi];
    float acc[kMaxAcc];
#pragma unroll
    for (int x = 0; x < kMaxAcc; ++x) acc[x] = 0.f;
    for (int b = gd.b0; b < gd.b1;) {
      const BlockDesc h = blocks[b];
      const int len = h.pad;
      switch (h.ij) {
        TCG_IJR(0, 1) TCG_IJR(0, 2) TCG_IJR(0, 3) TCG_IJR(0, 4) TCG_IJR(0, 5) TCG_IJR(0, 6)
        TCG_IJR(1, 0) TCG_IJR(1, 1) TCG_IJR(1, 2) TCG_IJR(1, 3) TCG_IJR(1, 4) TCG_IJR(1, 5)
        TCG_IJR(2, 0) TCG_IJR(2, 1) TCG_IJR(2, 2) TCG_IJR(2, 3) TCG_IJR(2, 4)
        TCG_IJR(3, 0) TCG_IJR(3, 1) TCG_IJR(3, 2) TCG_IJR(3, 3)
        TCG_IJR(4, 0) TCG_IJR(4, 1) TCG_IJR(4, 2)
        TCG_IJR(5, 0) TCG_IJR(5, 1)
        TCG_IJR(6, 0) TCG_IJR(0, 0)
        default: break;
      }
      b += len;
    }
    if (v >= 0) {
      const int cnt = cbin_rt<kH1>(gd.s1);
#pragma unroll
      for (int x = 0; x < kMaxAcc; ++x)
        if (x < cnt) {
          const int col = gd.out_off + x;
          out[om ? panel_offset(Cout, n, v, __ldg(om + col)) : panel_offset(Ws, n, v, col)] = acc[x];
        }
    }
    if (lane == 0) gi = atomicAdd(&next_group, 1);
    gi = __shfl_sync(0xffffffffu, gi, 0);
  }
}
// --------------------------------------------- TMA-staged blocked eMA
// ema_rt_blocked as a PERSISTENT kernel whose tile staging runs on the TMA
// engine: while the CTA computes tile t from the transposed [column][33]
// buffers, the rows of tile t + gridDim.x are already in flight as
// cp.async.bulk copies (SASS UBLKCP; one 16 B-aligned bulk copy per
// (vertex, panel) row, completion on an mbarrier's transaction count) into a
// row-major raw buffer.  The next iteration only transposes raw -> [col][33]
// through the per-colour maps (conflict-free reads: lanes walk consecutive
// columns of one vertex), so the HBM latency of staging is hidden behind the
// previous tile's FMAs instead of stalling the CTA.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// issue the bulk copies of tile t's rows (A then P, every panel of every
// vertex) into raw[v][RA + RP]; one thread arms the barrier first
__device__ __forceinline__ void rt_issue_tile(const float* __restrict__ Am, int Ca, const float* __restrict__ Pm,
                                              int Cpt, int32_t n, const int32_t* vids, int cnt, float* raw,
                                              int RS, int RA, uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  const int pa = num_panels(Ca), za = last_panel_width(Ca), pp = num_panels(Cpt), zp = last_panel_width(Cpt);
  if (lane == 0) {
    const uint32_t per_v = 4u * static_cast<uint32_t>((pa - 1) * kZ + za + (pp - 1) * kZ + zp);
    mbar_expect_tx(bar, per_v * static_cast<uint32_t>(cnt));
  }
  __syncwarp();
  if (lane < cnt) {
    const int64_t v = vids[lane];
    float* r = raw + static_cast<int64_t>(lane) * RS;
    for (int p = 0; p < pa; ++p) {
      const int zw = p == pa - 1 ? za : kZ;
      bulk_g2s(r + p * kZ, Am + static_cast<int64_t>(p) * n * kZ + v * zw, 4u * zw, bar);
    }
    for (int p = 0; p < pp; ++p) {
      const int zw = p == pp - 1 ? zp : kZ;
      bulk_g2s(r + RA + p * kZ, Pm + static_cast<int64_t>(p) * n * kZ + v * zw, 4u * zw, bar);
    }
  }
}

constexpr int kRtTmaThreads = 512;
__global__ void __launch_bounds__(kRtTmaThreads, 1)
ema_rt_blocked_tma(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca,
                   const float* __restrict__ Pm, int Cpt, const int32_t* __restrict__ pmap, int Wp,
                   const int32_t* __restrict__ vsorted, const int4* __restrict__ tiles, int ntiles,
                   const GroupDesc* __restrict__ groups, int ngroups, const BlockDesc* __restrict__ blocks, int Ws,
                   const int32_t* __restrict__ omap, int Cout, int32_t n, float* __restrict__ out, int RS, int RA) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int next_group;
  __shared__ int32_t vids[2][32];
  __shared__ int4 tinfo[2];
  float* raw = smem;                                // [32][RS], RS multiple of 32 floats
  float* sA = smem + 32 * RS;                       // [Wa][33]
  float* sP = sA + Wa * kSpitch;                    // [Wp][33]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  auto load_tile = [&](int t, int buf) {            // tile t's info and vertex ids (warp 0)
    const int4 ti = t < ntiles ? tiles[t] : make_int4(-1, 0, 0, 0);
    if (lane == 0) tinfo[buf] = ti;
    vids[buf][lane] = (ti.x >= 0 && lane < ti.z) ? vsorted[ti.y + lane] : -1;
    __syncwarp();
  };
  uint32_t phase = 0;
  int t = blockIdx.x, buf = 0;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // skip unused tiles (color -1) up front: they are numbered last per color
  if (warp == 0) {
    load_tile(t, 0);
    if (t < ntiles && tinfo[0].x >= 0) rt_issue_tile(Am, Ca, Pm, Cpt, n, vids[0], tinfo[0].z, raw, RS, RA, &bar);
  }
  __syncthreads();
  while (t < ntiles) {
    const int4 ti = tinfo[buf];
    const int tn = t + gridDim.x;
    if (ti.x >= 0) {
      mbar_wait(&bar, phase);
      phase ^= 1u;
      // transpose raw -> [col][33] through the colour's maps (every relabeled
      // row has exactly one storage column, so each row is rewritten; lanes of
      // missing vertices are never written out)
      const int c = ti.x;
      const int32_t* am = amap ? amap + static_cast<int64_t>(c) * Ca : nullptr;
      const int32_t* pm = pmap + static_cast<int64_t>(c) * Cpt;
      for (int v = warp; v < ti.z; v += nw) {
        const float* r = raw + static_cast<int64_t>(v) * RS;
        for (int col = lane; col < Ca; col += 32) {
          const int m = am ? __ldg(am + col) : (col < Wa ? col : -1);
          if (m >= 0) sA[m * kSpitch + v] = r[col];
        }
        for (int col = lane; col < Cpt; col += 32) {
          const int m = __ldg(pm + col);
          if (m >= 0) sP[m * kSpitch + v] = r[RA + col];
        }
      }
      if (threadIdx.x == 0) next_group = nw;
    }
    __syncthreads();  // raw consumed, sA/sP ready
    // prefetch the next tile's rows on the TMA engine while this one computes
    if (warp == 0) {
      load_tile(tn, buf ^ 1);
      if (tn < ntiles && tinfo[buf ^ 1].x >= 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        rt_issue_tile(Am, Ca, Pm, Cpt, n, vids[buf ^ 1], tinfo[buf ^ 1].z, raw, RS, RA, &bar);
      }
    }
    if (ti.x >= 0) {
      const int64_t v = vids[buf][lane];
      const int32_t* om = omap ? omap + static_cast<int64_t>(ti.x) * Ws : nullptr;
      for (int gi = warp; gi < ngroups;) {
        const GroupDesc gd = groups[gi];
        float acc[kMaxAcc];
#pragma unroll
        for (int x = 0; x < kMaxAcc; ++x) acc[x] = 0.f;
        for (int b = gd.b0; b < gd.b1;) {
          const BlockDesc h = blocks[b];
          const int len = h.pad;
          switch (h.ij) {
            TCG_IJR(0, 1) TCG_IJR(0, 2) TCG_IJR(0, 3) TCG_IJR(0, 4) TCG_IJR(0, 5) TCG_IJR(0, 6)
            TCG_IJR(1, 0) TCG_IJR(1, 1) TCG_IJR(1, 2) TCG_IJR(1, 3) TCG_IJR(1, 4) TCG_IJR(1, 5)
            TCG_IJR(2, 0) TCG_IJR(2, 1) TCG_IJR(2, 2) TCG_IJR(2, 3) TCG_IJR(2, 4)
            TCG_IJR(3, 0) TCG_IJR(3, 1) TCG_IJR(3, 2) TCG_IJR(3, 3)
            TCG_IJR(4, 0) TCG_IJR(4, 1) TCG_IJR(4, 2)
            TCG_IJR(5, 0) TCG_IJR(5, 1)
            TCG_IJR(6, 0) TCG_IJR(0, 0)
            default: break;
          }
          b += len;
        }
        if (v >= 0) {
          const int cnt = cbin_rt<kH1>(gd.s1);
#pragma unroll
          for (int x = 0; x < kMaxAcc; ++x)
            if (x < cnt) {
              const int col = gd.out_off + x;
              out[om ? panel_offset(Cout, n, v, __ldg(om + col)) : panel_offset(Ws, n, v, col)] = acc[x];
            }
        }
        if (lane == 0) gi = atomicAdd(&next_group, 1);
        gi = __shfl_sync(0xffffffffu, gi, 0);
      }
    }
    __syncthreads();  // sA/sP free for the next transpose
    t = tn;
    buf ^= 1;
  }
}
// ------------------------------------ warp-specialized pipelined blocked eMA
// ema_rt_blocked as a persistent, warp-specialized pipeline (the SM's smem
// holds TWO transposed tiles, 2 x (Wa + Wp) x 33 floats):
//   * warp 16 (producer) stages tile i + 2 into the buffer tile i used, the
//     moment every output group of tile i is done (mbarrier `empty`), with
//     4-byte cp.async copies (SASS LDGSTS) straight into the [column][33]
//     layout through the per-colour maps -- no registers, no transpose pass;
//     `full` completes when those copies land (cp.async.mbarrier.arrive);
//   * warps 0-15 (consumers) take (tile, group) items from ONE queue that runs
//     across tile boundaries, so a warp that finishes tile i's last group moves
//     on to tile i+1 instead of waiting at a CTA barrier (the tail that made
//     the TMA variant slow), and never waits for HBM unless the producer is
//     two tiles behind.
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kRtPipeConsumers = 12;  // consumer warps (>= 1 output group each per tile)
constexpr int kRtPipeProducers = 8;   // producer warps: bytes in flight (one warp alone keeps too few)
template <int NP, int NC>
__global__ void __launch_bounds__((NP + NC) * 32, 1)
ema_rt_blocked_pipe(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca,
                    const float* __restrict__ Pm, int Cpt, const int32_t* __restrict__ pmap, int Wp,
                    const int32_t* __restrict__ vsorted, const int4* __restrict__ tiles, int ntiles,
                    const GroupDesc* __restrict__ groups, int ngroups, const BlockDesc* __restrict__ blocks, int Ws,
                    const int32_t* __restrict__ omap, int Cout, int32_t n, float* __restrict__ out) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  __shared__ int32_t vids[2][32];
  __shared__ int4 tinfo[2];
  __shared__ int next_item, ntile_cta;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bufsz = (Wa + Wp) * kSpitch;
  if (threadIdx.x == 0) {
    mbar_init(&full[0], NP);
    mbar_init(&full[1], NP);
    mbar_init(&empty[0], static_cast<uint32_t>(ngroups));
    mbar_init(&empty[1], static_cast<uint32_t>(ngroups));
    next_item = 0;
  }
  if (warp == 0) {  // this CTA's tiles blockIdx.x + i * gridDim.x that hold vertices (a prefix)
    int cnt = 0;
    for (int i0 = 0;; i0 += 32) {
      const int t = blockIdx.x + (i0 + lane) * static_cast<int>(gridDim.x);
      const bool ok = t < ntiles && tiles[t].x >= 0;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      cnt += __popc(m);
      if (m != 0xffffffffu) break;
    }
    if (lane == 0) ntile_cta = cnt;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int nt = ntile_cta;
  if (warp >= NC) {
    // ----------------------------------------------------------- producers
    const int pw = warp - NC;
    for (int i = 0; i < nt; ++i) {
      const int b = i & 1;
      if (i >= 2) mbar_wait(&empty[b], static_cast<uint32_t>(((i >> 1) - 1) & 1));  // tile i-2 fully consumed
      const int t = blockIdx.x + i * static_cast<int>(gridDim.x);
      const int4 ti = tiles[t];
      const int vid = lane < ti.z ? vsorted[ti.y + lane] : -1;
      if (pw == 0) {
        if (lane == 0) tinfo[b] = ti;
        vids[b][lane] = vid;
      }
      float* sA = smem + b * bufsz;
      float* sP = sA + Wa * kSpitch;
      const int32_t* am = amap ? amap + static_cast<int64_t>(ti.x) * Ca : nullptr;
      const int32_t* pm = pmap + static_cast<int64_t>(ti.x) * Cpt;
      // lane = column (consecutive columns of one vertex row: coalesced
      // reads); producer warp pw takes column chunks pw, pw + NP, ...
      for (int c0 = pw * 32; c0 < Ca; c0 += NP * 32) {
        const int c = c0 + lane;
        const int m = c < Ca ? (am ? __ldg(am + c) : (c < Wa ? c : -1)) : -1;
        const int p = c / kZ, zw = panel_width(Ca, p);
        const float* src = Am + static_cast<int64_t>(p) * n * kZ + (c % kZ);
        for (int v = 0; v < ti.z; ++v) {
          const int64_t u = __shfl_sync(0xffffffffu, vid, v);
          if (m >= 0) cp_async4(sA + m * kSpitch + v, src + u * zw);
        }
      }
      for (int c0 = pw * 32; c0 < Cpt; c0 += NP * 32) {
        const int c = c0 + lane;
        const int m = c < Cpt ? __ldg(pm + c) : -1;
        const int p = c / kZ, zw = panel_width(Cpt, p);
        const float* src = Pm + static_cast<int64_t>(p) * n * kZ + (c % kZ);
        for (int v = 0; v < ti.z; ++v) {
          const int64_t u = __shfl_sync(0xffffffffu, vid, v);
          if (m >= 0) cp_async4(sP + m * kSpitch + v, src + u * zw);
        }
      }
      cp_async_arrive(&full[b]);  // pending +1 now, -1 when this lane's copies land
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[b]);  // this warp's expected arrival (vids / tinfo written)
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const int total = nt * ngroups;
  int item = 0;
  if (lane == 0) item = atomicAdd(&next_item, 1);
  item = __shfl_sync(0xffffffffu, item, 0);
  while (item < total) {
    const int i = item / ngroups, gi = item - i * ngroups;
    const int b = i & 1;
    mbar_wait(&full[b], static_cast<uint32_t>((i >> 1) & 1));
    const float* sA = smem + b * bufsz;
    const float* sP = sA + Wa * kSpitch;
    const int4 ti = tinfo[b];
    const int64_t v = vids[b][lane];
    const int32_t* om = omap ? omap + static_cast<int64_t>(ti.x) * Ws : nullptr;
    const GroupDesc gd = groups[gi];
    float acc[kMaxAcc];
#pragma unroll
    for (int x = 0; x < kMaxAcc; ++x) acc[x] = 0.f;
    for (int bb = gd.b0; bb < gd.b1;) {
      const BlockDesc h = blocks[bb];
      const int len = h.pad;
      const int b = bb;
      switch (h.ij) {
        TCG_IJR(0, 1) TCG_IJR(0, 2) TCG_IJR(0, 3) TCG_IJR(0, 4) TCG_IJR(0, 5) TCG_IJR(0, 6)
        TCG_IJR(1, 0) TCG_IJR(1, 1) TCG_IJR(1, 2) TCG_IJR(1, 3) TCG_IJR(1, 4) TCG_IJR(1, 5)
        TCG_IJR(2, 0) TCG_IJR(2, 1) TCG_IJR(2, 2) TCG_IJR(2, 3) TCG_IJR(2, 4)
        TCG_IJR(3, 0) TCG_IJR(3, 1) TCG_IJR(3, 2) TCG_IJR(3, 3)
        TCG_IJR(4, 0) TCG_IJR(4, 1) TCG_IJR(4, 2)
        TCG_IJR(5, 0) TCG_IJR(5, 1)
        TCG_IJR(6, 0) TCG_IJR(0, 0)
        default: break;
      }
      bb += len;
    }
    if (v >= 0) {
      const int cnt = cbin_rt<kH1>(gd.s1);
#pragma unroll
      for (int x = 0; x < kMaxAcc; ++x)
        if (x < cnt) {
          const int col = gd.out_off + x;
          out[om ? panel_offset(Cout, n, v, __ldg(om + col)) : panel_offset(Ws, n, v, col)] = acc[x];
        }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty[b]);  // one of the tile's ngroups items done (its smem reads are complete)
      item = atomicAdd(&next_item, 1);
    }
    item = __shfl_sync(0xffffffffu, item, 0);
  }
}

#undef TCG_IJR

// Root on a same-color tile: fp64 dot product over the C(k-1, a-1) splits of
// the (k-1) colors (ALEAF: the single P value).  Per-vertex totals to
// root_out[v]; fixed-order per-tile totals (0 for unused tiles).
template <bool ALEAF>
__global__ void __launch_bounds__(kEmaWarps * 32)
ema_rt_root(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca, const float* __restrict__ Pm, int Cpt,
            const int32_t* __restrict__ pmap, int Wp, const int32_t* __restrict__ vsorted,
            const int4* __restrict__ tiles, const int2* __restrict__ split, int pairs, int32_t n,
            double* __restrict__ root_out, double* __restrict__ root_acc, double* __restrict__ tile_tot) {
  extern __shared__ float smem[];
  __shared__ double red[kEmaWarps][kTileV];
  __shared__ int32_t vids[32];
  const int4 tile = tiles[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (tile.x < 0) {
    if (threadIdx.x == 0) tile_tot[blockIdx.x] = 0.0;
    return;
  }
  const int c = tile.x;
  if (threadIdx.x < 32) vids[threadIdx.x] = static_cast<int>(threadIdx.x) < tile.z ? vsorted[tile.y + threadIdx.x] : -1;
  __syncthreads();
  float* sA = smem;
  float* sP = smem + (ALEAF ? 0 : Wa * kSpitch);
  if (!ALEAF) stage_rows<4>(Am, Ca, n, vids, sA, amap ? amap + static_cast<int64_t>(c) * Ca : nullptr);
  stage_rows<4>(Pm, Cpt, n, vids, sP, pmap + static_cast<int64_t>(c) * Cpt);
  __syncthreads();
  double acc = 0;
  if (ALEAF) {
    if (warp == 0) acc = static_cast<double>(sP[lane]);
  } else {
    for (int p = warp; p < pairs; p += nw) {
      const int2 s = __ldg(split + p);
      acc = fma(static_cast<double>(sA[s.x * kSpitch + lane]), static_cast<double>(sP[s.y * kSpitch + lane]), acc);
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    double tot = 0;
    for (int w = 0; w < nw; ++w) tot += red[w][lane];
    const int v = vids[lane];
    if (v >= 0) {
      root_out[v] = tot;
      if (root_acc) root_acc[v] += tot;
    } else {
      tot = 0;
    }
    for (int o = 16; o; o >>= 1) tot += __shfl_down_sync(0xffffffffu, tot, o);
    if (lane == 0) tile_tot[blockIdx.x] = tot;
  }
}

// Streamed active-leaf epilogue: one group's finished P' columns (n x Ct
// scratch, columns [0, fpad)) -> M_s[v, emap[c(v)][col]] (RR column or RS
// slot; -1 = the set contains c(v), dropped).
__global__ void __launch_bounds__(256)
pstream_copy(const float* __restrict__ Tg, int Ct, int fpad, const int32_t* __restrict__ emap, int Cps,
             const uint8_t* __restrict__ colors, int Cout, int32_t n, float* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(n) * fpad;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i / fpad;
    const int col = static_cast<int>(i - v * fpad);
    const int oc = __ldg(emap + static_cast<int64_t>(colors[v]) * Cps + col);
    if (oc >= 0) out[panel_offset(Cout, n, v, oc)] = Tg[panel_offset(Ct, n, v, col)];
  }
}

// ------------------------------------------- vertex-per-CTA rooted eMA
// Nodes whose 32-vertex tile does not fit in shared memory (k = 15/17: cfg5
// node 1 stages C(16,7) + C(16,4) floats per vertex) run the rooted (k-1)
// problem one vertex per CTA: the vertex's RR active row and its P' row,
// mapped to relabeled indices through the vertex color's pmap, are staged
// contiguously in smem and the threads split the output groups of the
// register-blocked descriptors (build_blocked(k-1, s-1, a-1)).  a/k of the
// full-table FMAs, s/k of its table bytes.

// P' row of vertex v (Cpt storage columns) -> dst[pm[col]] (relabeled index;
// -1: the column contains the vertex color and is never used)
__device__ __forceinline__ void stage_row_pmap(const float* __restrict__ T, int Cpt, int32_t n, int64_t v,
                                               float* dst, const int32_t* __restrict__ pm) {
  const int panels = num_panels(Cpt);
  const int zl = last_panel_width(Cpt);
  const int total4 = ((panels - 1) * kZ + zl) / 4;
  for (int f = threadIdx.x; f < total4; f += blockDim.x) {
    const int c0 = f * 4;
    if (c0 >= Cpt) continue;
    const int p = c0 / kZ, z4 = c0 % kZ;
    const int zw = p == panels - 1 ? zl : kZ;
    const float4 x = __ldg(reinterpret_cast<const float4*>(T + static_cast<int64_t>(p) * n * kZ + v * zw + z4));
    const int m0 = __ldg(pm + c0);
    const int m1 = c0 + 1 < Cpt ? __ldg(pm + c0 + 1) : -1;
    const int m2 = c0 + 2 < Cpt ? __ldg(pm + c0 + 2) : -1;
    const int m3 = c0 + 3 < Cpt ? __ldg(pm + c0 + 3) : -1;
    if (m0 >= 0) dst[m0] = x.x;
    if (m1 >= 0) dst[m1] = x.y;
    if (m2 >= 0) dst[m2] = x.z;
    if (m3 >= 0) dst[m3] = x.w;
  }
}

// stage_row with cp.async (LDGSTS.128): the copies of a thread are all in flight at once and
// hold no registers; the caller waits with cp_async_wait_all() before its barrier.
__device__ __forceinline__ void stage_row_async(const float* __restrict__ T, int C, int32_t n, int64_t v, float* dst) {
  const int panels = num_panels(C);
  const int zl = last_panel_width(C);
  const int total4 = ((panels - 1) * kZ + zl) / 4;
  const uint32_t d0 = smem_u32(dst);
  for (int f = threadIdx.x; f < total4; f += blockDim.x) {
    const int p = (f * 4) / kZ, z4 = (f * 4) % kZ;
    const int zw = p == panels - 1 ? zl : kZ;
    const float* src = T + static_cast<int64_t>(p) * n * kZ + v * zw + z4;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d0 + f * 16), "l"(src) : "memory");
  }
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---- H-colour register blocking (H = 6/7/8), generic over H: the
// H1-subset micro-patterns (i, j) of build_blocked(k', s', a', H), pattern
// code i * 16 + j.  Triples (a1, p1, a1|p1) of a pattern are one constexpr
// table per (H, i, j).
template <int H, int I, int J>
struct TripTab {
  static constexpr int NT = cbin(H, I) * cbin(H - I, J);
  struct Arr { Trip t[NT > 0 ? NT : 1]; };
  static constexpr int rank(unsigned m) {
    int idx = 0, pos = 0;
    for (int c = 0; c < H; ++c)
      if (m >> c & 1u) idx += cbin(c, ++pos);
    return idx;
  }
  static constexpr Arr make() {
    Arr r{};
    int n = 0;
    for (unsigned am = 0; am < (1u << H); ++am) {
      if (cpop(am) != I) continue;
      for (unsigned pm = 0; pm < (1u << H); ++pm)
        if (cpop(pm) == J && !(am & pm)) r.t[n++] = Trip{rank(am), rank(pm), rank(am | pm)};
    }
    return r;
  }
  static constexpr Arr tab = make();
};

template <int H, int I, int J, int... T>
__device__ __forceinline__ void micro_fma_h(const float* a, const float* p, float* acc,
                                            std::integer_sequence<int, T...>) {
  ((acc[TripTab<H, I, J>::tab.t[T].o] =
        fmaf(a[TripTab<H, I, J>::tab.t[T].a], p[TripTab<H, I, J>::tab.t[T].p], acc[TripTab<H, I, J>::tab.t[T].o])),
   ...);
}

// shared-memory word at a 32-bit shared address plus a compile-time byte
// offset (explicit ld.shared: the generic-pointer form recomputes the shared
// window base and the row stride for every block)
template <int OFF>
__device__ __forceinline__ float lds_imm(uint32_t addr) {
  float v;
  asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
  return v;
}
template <int N, int... X>
__device__ __forceinline__ void lds_row(float (&dst)[N], uint32_t addr, std::integer_sequence<int, X...>) {
  ((dst[X] = lds_imm<X * 4>(addr)), ...);
}

template <int H, int I, int J>
__device__ __forceinline__ void micro_block_h(uint32_t sa, uint32_t sp, float* acc) {
  if constexpr (I + J <= H) {
    constexpr int NA = cbin(H, I), NP = cbin(H, J);
    float a[NA], p[NP];
    lds_row(a, sa, std::make_integer_sequence<int, NA>{});
    lds_row(p, sp, std::make_integer_sequence<int, NP>{});
    micro_fma_h<H, I, J>(a, p, acc, std::make_integer_sequence<int, TripTab<H, I, J>::NT>{});
  }
}

// dense pattern code of (i, j), i + j <= 8, in TCG_HCASES order (a dense switch
// compiles to one indexed branch)
__host__ __device__ constexpr int hcode(int i, int j) { return i * 9 - i * (i - 1) / 2 + j; }

// one run of blocks with the same pattern (I, J).  The task's descriptors
// {a_off | p_off << 16} form one linear stream of 32-word chunks (32 / gpt
// block steps each); lane l holds word l of the current chunk and of the two
// chunks after it (loaded two chunks -- >= 4 blocks -- ahead: the stream
// lives in L2), and a block's descriptor is a shuffle away.  Not unrolled:
// the 45 pattern bodies already exceed the instruction cache.
#define TCG_HC(I, J)                                                                 \
  case hcode(I, J): {                                                                \
    _Pragma("unroll 1")                                                              \
    for (int q = 0; q < len; ++q) {                                                  \
      const uint32_t d = __shfl_sync(0xffffffffu, cur, sc + gl);                     \
      sc += gpt;                                                                     \
      if (sc == 32) {                                                                \
        sc = 0;                                                                      \
        cur = n1;                                                                    \
        n1 = n2;                                                                     \
        wo += 32;                                                                    \
        n2 = __ldg(blocks + wo);                                                     \
      }                                                                              \
      micro_block_h<H, I, J>((d & 0xFFFFu) * 4u + aA, (d >> 16) * 4u + aP, acc);     \
    }                                                                                \
  } break;
#define TCG_HCASES                                                                                        \
  TCG_HC(0, 0) TCG_HC(0, 1) TCG_HC(0, 2) TCG_HC(0, 3) TCG_HC(0, 4) TCG_HC(0, 5) TCG_HC(0, 6) TCG_HC(0, 7) \
  TCG_HC(0, 8) TCG_HC(1, 0) TCG_HC(1, 1) TCG_HC(1, 2) TCG_HC(1, 3) TCG_HC(1, 4) TCG_HC(1, 5) TCG_HC(1, 6) \
  TCG_HC(1, 7) TCG_HC(2, 0) TCG_HC(2, 1) TCG_HC(2, 2) TCG_HC(2, 3) TCG_HC(2, 4) TCG_HC(2, 5) TCG_HC(2, 6) \
  TCG_HC(3, 0) TCG_HC(3, 1) TCG_HC(3, 2) TCG_HC(3, 3) TCG_HC(3, 4) TCG_HC(3, 5) TCG_HC(4, 0) TCG_HC(4, 1) \
  TCG_HC(4, 2) TCG_HC(4, 3) TCG_HC(4, 4) TCG_HC(5, 0) TCG_HC(5, 1) TCG_HC(5, 2) TCG_HC(5, 3) TCG_HC(6, 0) \
  TCG_HC(6, 1) TCG_HC(6, 2) TCG_HC(7, 0) TCG_HC(7, 1) TCG_HC(8, 0)

// V vertices per pass (staged at strides sa/sp floats, == 32/V mod 32 so the
// V lanes sharing a group hit different banks).  A TASK is 32/V output groups
// of one shape (the same sequence of pattern runs, host build_rtv_tasks) x V
// vertices: the warp walks ONE run list (uniform pattern dispatch, no
// divergence), and only the operand offsets differ per lane -- one packed
// 4 B descriptor {a_off | p_off << 16} per (block step, group), stored
// step-major so a warp reads its task's descriptors as coalesced 128 B chunks.  The host orders
// each group's blocks inside a run so that the groups' offsets of a step fall
// on different banks (residues mod 32/V distinct where possible).  Warps take
// tasks from a per-pass queue, largest first.
struct RtvTask {
  int32_t blk0, run0, nruns, s1;
};

constexpr int kRtvThreads = 448;  // 2 CTAs x 14 warps per SM at 72 registers
template <int H, int THREADS>
__global__ void __launch_bounds__(THREADS, THREADS > 512 ? 1 : 2)
ema_rtv_blocked(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca, const float* __restrict__ Pm, int Cpt,
                const int32_t* __restrict__ pmap, const uint8_t* __restrict__ colors,
                const RtvTask* __restrict__ tasks, int ntasks, const int32_t* __restrict__ gout,
                const uint32_t* __restrict__ runs, const uint32_t* __restrict__ blocks, int Ws,
                const int32_t* __restrict__ omap, int Cout, int32_t n, float* __restrict__ out, int V, int sa,
                int sp) {
  constexpr int kAcc = cbin(H, H / 2);
  extern __shared__ float smem[];
  __shared__ int next_task;
  float* sP0 = smem + V * sa;
  const int lane = threadIdx.x & 31;
  const int gpt = 32 / V;
  const int gl = lane / V, j = lane - gl * V;
  const uint32_t aA = smem_u32(smem + j * sa), aP = smem_u32(sP0 + j * sp);  // the lane's vertex rows
  for (int64_t v0 = static_cast<int64_t>(blockIdx.x) * V; v0 < n; v0 += static_cast<int64_t>(gridDim.x) * V) {
    __syncthreads();
    if (threadIdx.x == 0) next_task = blockDim.x >> 5;
    for (int jj = 0; jj < V && v0 + jj < n; ++jj) {
      if (amap) stage_row_pmap(Am, Ca, n, v0 + jj, smem + jj * sa, amap + static_cast<int64_t>(colors[v0 + jj]) * Ca);
      else stage_row_async(Am, Wa, n, v0 + jj, smem + jj * sa);
      stage_row_pmap(Pm, Cpt, n, v0 + jj, sP0 + jj * sp, pmap + static_cast<int64_t>(colors[v0 + jj]) * Cpt);
    }
    cp_async_wait_all();
    __syncthreads();
    const int64_t v = v0 + j;
    for (int task = threadIdx.x >> 5; task < ntasks;) {
      const int4 t = __ldg(reinterpret_cast<const int4*>(tasks) + task);  // {blk0, run0, nruns, s1}
      const int out_off = __ldg(gout + task * gpt + gl);
      float acc[kAcc];
#pragma unroll
      for (int x = 0; x < kAcc; ++x) acc[x] = 0.f;
      uint32_t wo = static_cast<uint32_t>(t.x) + lane + 64;  // (the lane's word of the chunk loaded last)
      uint32_t cur = __ldg(blocks + wo - 64), n1 = __ldg(blocks + wo - 32), n2 = __ldg(blocks + wo);
      int sc = 0;                                     // first word of the current step in the chunk
      uint32_t rr = __ldg(runs + t.y);
      for (int r = 0; r < t.z; ++r) {
        const uint32_t rn = r + 1 < t.z ? __ldg(runs + t.y + r + 1) : 0u;
        const int len = static_cast<int>(rr >> 8);
        switch (rr & 0xFFu) {
          TCG_HCASES
          default: break;
        }
        rr = rn;
      }
      if (out_off >= 0 && v < n) {
        const int32_t* om = omap ? omap + static_cast<int64_t>(colors[v]) * Ws : nullptr;
        const int cnt = cbin_rt<H>(t.w);
#pragma unroll
        for (int x = 0; x < kAcc; ++x)
          if (x < cnt) {
            const int col = out_off + x;
            out[om ? panel_offset(Cout, n, v, __ldg(om + col)) : panel_offset(Ws, n, v, col)] = acc[x];
          }
      }
      if (lane == 0) task = atomicAdd(&next_task, 1);
      task = __shfl_sync(0xffffffffu, task, 0);
    }
  }
}
#undef TCG_HC
#undef TCG_HCASES

// Root, one vertex per CTA: fp64 dot product over the relabeled split pairs,
// fixed-order reduction (shuffle tree inside a warp, then the warps in order;
// three barriers per vertex) -> root_out[v] (root_reduce then sums root_out).
__global__ void __launch_bounds__(256)
ema_rtv_root(const float* __restrict__ Am, int Wa, const int32_t* __restrict__ amap, int Ca, const float* __restrict__ Pm, int Cpt,
             const int32_t* __restrict__ pmap, const uint8_t* __restrict__ colors, const int2* __restrict__ split,
             int pairs, int32_t n, double* __restrict__ root_out, double* __restrict__ root_acc) {
  extern __shared__ float smem[];
  __shared__ double red[8];
  float* sA = smem;
  float* sP = smem + row_floats(Wa);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
    const int c = colors[v];
    __syncthreads();
    if (amap) stage_row_pmap(Am, Ca, n, v, sA, amap + static_cast<int64_t>(c) * Ca);
    else stage_row_async(Am, Wa, n, v, sA);
    stage_row_pmap(Pm, Cpt, n, v, sP, pmap + static_cast<int64_t>(c) * Cpt);
    cp_async_wait_all();
    __syncthreads();
    double acc = 0;
    for (int p = threadIdx.x; p < pairs; p += blockDim.x) {
      const int2 s = __ldg(split + p);
      acc = fma(static_cast<double>(sA[s.x]), static_cast<double>(sP[s.y]), acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < 8; ++w) t += red[w];
      root_out[v] = t;
      if (root_acc) root_acc[v] += t;
    }
  }
}

}  // namespace dev
}  // namespace tcg
