// host.cpp -- host-side subsystems (see host.hpp for the reference mapping).
#include "host.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <condition_variable>
#include <mutex>
#include <thread>

namespace tcg {

// ----------------------------------------------------------------- threads
int host_threads() {
  static const int t = [] {
    unsigned h = std::thread::hardware_concurrency();
    return static_cast<int>(h ? std::min(h, 64u) : 4u);
  }();
  return t;
}

// fn(begin, end, worker) over [0, total) in T static slices
void parallel_for(int64_t total, const std::function<void(int64_t, int64_t, int)>& fn) {
  const int T = static_cast<int>(std::min<int64_t>(host_threads(), std::max<int64_t>(1, total / 4096)));
  if (T <= 1) { fn(0, total, 0); return; }
  std::vector<std::thread> th;
  for (int w = 0; w < T; ++w)
    th.emplace_back([&, w] { fn(total * w / T, total * (w + 1) / T, w); });
  for (auto& t : th) t.join();
}

// dynamic chunks (for skewed per-row work such as hub rows)
static void parallel_chunks(int64_t total, int64_t chunk, const std::function<void(int64_t, int64_t)>& fn) {
  std::atomic<int64_t> next{0};
  const int T = static_cast<int>(std::min<int64_t>(host_threads(), std::max<int64_t>(1, total / chunk)));
  auto body = [&] {
    for (;;) {
      int64_t b = next.fetch_add(chunk);
      if (b >= total) return;
      fn(b, std::min(total, b + chunk));
    }
  };
  if (T <= 1) { body(); return; }
  std::vector<std::thread> th;
  for (int w = 0; w < T; ++w) th.emplace_back(body);
  for (auto& t : th) t.join();
}

// ------------------------------------------------------------- MT19937-64
Mt64::Mt64(uint64_t seed) {
  x[0] = seed;
  for (int j = 1; j < 312; ++j) x[j] = 6364136223846793005ULL * (x[j - 1] ^ (x[j - 1] >> 62)) + j;
  i = 312;
}

void Mt64::twist() {
  constexpr uint64_t U = 0xFFFFFFFF80000000ULL, L = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  int j = 0;
  for (; j < 156; ++j) {
    const uint64_t y = (x[j] & U) | (x[j + 1] & L);
    x[j] = x[j + 156] ^ (y >> 1) ^ ((y & 1) * A);
  }
  for (; j < 311; ++j) {
    const uint64_t y = (x[j] & U) | (x[j + 1] & L);
    x[j] = x[j - 156] ^ (y >> 1) ^ ((y & 1) * A);
  }
  const uint64_t y = (x[311] & U) | (x[0] & L);
  x[311] = x[155] ^ (y >> 1) ^ ((y & 1) * A);
  i = 0;
}

// ------------------------------------------------------------------- graph
int32_t Csr::max_degree() const {
  int64_t best = 0;
  for (int32_t v = 0; v < n; ++v) best = std::max(best, row_ptr[v + 1] - row_ptr[v]);
  return static_cast<int32_t>(best);
}

// Counting-sort CSR build: scatter both directions of every non-loop edge
// into per-row slots, then sort + dedup each row in parallel.  Same output
// as from_edges (graph.hpp:65-95): symmetric union, no self-loops, no
// duplicates, rows ascending.
Csr csr_from_edges(const int32_t* edges, int64_t m, int32_t n_hint) {
  int32_t n = n_hint;
  if (n < 0) {
    std::vector<int32_t> mx(host_threads(), -1);
    parallel_for(2 * m, [&](int64_t b, int64_t e, int w) {
      int32_t v = -1;
      for (int64_t j = b; j < e; ++j) v = std::max(v, edges[j]);
      mx[w] = std::max(mx[w], v);
    });
    n = *std::max_element(mx.begin(), mx.end()) + 1;
  }
  std::atomic<bool> bad{false};
  parallel_for(2 * m, [&](int64_t b, int64_t e, int) {
    for (int64_t j = b; j < e; ++j)
      if (edges[j] < 0 || edges[j] >= n) { bad = true; return; }
  });
  if (bad) throw parse_error("vertex id out of range [0, " + std::to_string(n) + ")");

  Csr g;
  g.n = n;
  std::vector<int64_t> cur(static_cast<size_t>(n) + 1, 0);
  parallel_for(m, [&](int64_t b, int64_t e, int) {
    for (int64_t j = b; j < e; ++j) {
      const int32_t u = edges[2 * j], v = edges[2 * j + 1];
      if (u == v) continue;
      __atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED);
      __atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED);
    }
  });
  std::vector<int64_t> start(static_cast<size_t>(n) + 1, 0);
  for (int32_t v = 0; v < n; ++v) start[v + 1] = start[v] + cur[v];
  std::memcpy(cur.data(), start.data(), sizeof(int64_t) * n);
  std::vector<int32_t> tmp(static_cast<size_t>(std::max<int64_t>(start[n], 1)));
  parallel_for(m, [&](int64_t b, int64_t e, int) {
    for (int64_t j = b; j < e; ++j) {
      const int32_t u = edges[2 * j], v = edges[2 * j + 1];
      if (u == v) continue;
      tmp[__atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED)] = v;
      tmp[__atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED)] = u;
    }
  });
  std::vector<int64_t> deg(static_cast<size_t>(n), 0);
  parallel_chunks(n, 4096, [&](int64_t b, int64_t e) {
    for (int64_t v = b; v < e; ++v) {
      int32_t* lo = tmp.data() + start[v];
      int32_t* hi = tmp.data() + start[v + 1];
      std::sort(lo, hi);
      deg[v] = std::unique(lo, hi) - lo;
    }
  });
  g.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int32_t v = 0; v < n; ++v) g.row_ptr[v + 1] = g.row_ptr[v] + deg[v];
  g.col.resize(static_cast<size_t>(g.row_ptr[n]));
  parallel_chunks(n, 16384, [&](int64_t b, int64_t e) {
    for (int64_t v = b; v < e; ++v)
      std::memcpy(g.col.data() + g.row_ptr[v], tmp.data() + start[v], sizeof(int32_t) * deg[v]);
  });
  return g;
}

Csr csr_adopt(int32_t n, const int64_t* row_ptr, const int32_t* col, bool check_symmetry) {
  if (n < 0 || !row_ptr || row_ptr[0] != 0) throw parse_error("bad CSR row_ptr");
  for (int32_t v = 0; v < n; ++v)
    if (row_ptr[v + 1] < row_ptr[v]) throw parse_error("CSR row_ptr not monotone");
  Csr g;
  g.n = n;
  g.row_ptr.assign(row_ptr, row_ptr + n + 1);
  g.col.assign(col, col + row_ptr[n]);
  std::atomic<int> bad{0};
  parallel_chunks(n, 4096, [&](int64_t b, int64_t e) {
    for (int64_t v = b; v < e && !bad; ++v) {
      for (int64_t j = g.row_ptr[v]; j < g.row_ptr[v + 1]; ++j) {
        const int32_t u = g.col[j];
        if (u < 0 || u >= n || u == v) { bad = 1; return; }
        if (j > g.row_ptr[v] && g.col[j - 1] >= u) { bad = 2; return; }
        if (check_symmetry &&
            !std::binary_search(g.col.data() + g.row_ptr[u], g.col.data() + g.row_ptr[u + 1],
                                static_cast<int32_t>(v))) { bad = 3; return; }
      }
    }
  });
  if (bad == 1) throw parse_error("CSR column out of range or self-loop");
  if (bad == 2) throw parse_error("CSR row not strictly ascending");
  if (bad == 3) throw parse_error("CSR not symmetric");
  return g;
}

// synthgen.hpp:40-74: one sequential MT stream, `scale` unit() draws per
// edge.  The stream is inherently serial, so it is pipelined: one producer
// thread runs only the 312-word twists and copies raw state blocks into a
// ring of chunks; worker threads temper, convert (Rng::unit) and descend the
// quadrants for whole edges (chunks are multiples of 312*scale words).
Csr generate_rmat(int scale, int64_t nedges, double a, double b, double c, double d,
                  uint64_t seed) {
  if (scale < 1 || scale > 26) throw invalid_argument("rmat scale must be in [1, 26]");
  if (nedges < 1) throw invalid_argument("rmat edge target must be >= 1");
  if (std::abs(a + b + c + d - 1.0) > 1e-9)
    throw invalid_argument("rmat quadrant probabilities must sum to 1");
  const int32_t n = static_cast<int32_t>(int64_t{1} << scale);
  std::vector<int32_t> e(static_cast<size_t>(2 * nedges));
  const double ab = a + b, abc = ab + c;
  const int64_t total_words = nedges * scale;
  const int64_t blocks_per_chunk = static_cast<int64_t>(scale) * 64;  // chunk = 312*scale*64 words
  const int64_t chunk_words = 312 * blocks_per_chunk;
  const int64_t nchunks = (total_words + chunk_words - 1) / chunk_words;
  const int workers = std::max(1, host_threads() - 1);
  const int ring = 2 * workers + 2;
  std::vector<std::vector<uint64_t>> buf(ring, std::vector<uint64_t>(chunk_words));
  std::vector<int64_t> slot_chunk(ring, -1);   // chunk held by the slot (-1 free)
  std::mutex mu;
  std::condition_variable cv_free, cv_ready;
  std::atomic<int64_t> next_chunk{0};

  auto consume = [&](int64_t ch, const uint64_t* raw) {
    const int64_t w0 = ch * chunk_words;
    const int64_t w1 = std::min(total_words, w0 + chunk_words);
    for (int64_t w = w0; w < w1; w += scale) {
      int32_t row = 0, cl = 0;
      for (int level = 0; level < scale; ++level) {
        uint64_t z = raw[w - w0 + level];
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        z ^= (z >> 43);
        const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
        const int32_t rb = u >= ab, cb = (u >= a && u < ab) || u >= abc;
        row = (row << 1) | rb;
        cl = (cl << 1) | cb;
      }
      e[2 * (w / scale)] = row;
      e[2 * (w / scale) + 1] = cl;
    }
  };
  std::thread producer([&] {
    Mt64 rng(seed);
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int slot = static_cast<int>(ch % ring);
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_free.wait(lk, [&] { return slot_chunk[slot] == -1; });
      }
      uint64_t* dst = buf[slot].data();
      const int64_t words = std::min(chunk_words, total_words - ch * chunk_words);
      for (int64_t o = 0; o < words; o += 312) {
        rng.twist();
        std::memcpy(dst + o, rng.x, sizeof(uint64_t) * std::min<int64_t>(312, words - o));
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        slot_chunk[slot] = ch;
      }
      cv_ready.notify_all();
    }
  });
  std::vector<std::thread> th;
  for (int t = 0; t < workers; ++t)
    th.emplace_back([&] {
      for (;;) {
        const int64_t ch = next_chunk.fetch_add(1);
        if (ch >= nchunks) return;
        const int slot = static_cast<int>(ch % ring);
        {
          std::unique_lock<std::mutex> lk(mu);
          cv_ready.wait(lk, [&] { return slot_chunk[slot] == ch; });
        }
        consume(ch, buf[slot].data());
        {
          std::lock_guard<std::mutex> lk(mu);
          slot_chunk[slot] = -1;
        }
        cv_free.notify_all();
      }
    });
  producer.join();
  for (auto& t : th) t.join();
  return csr_from_edges(e.data(), nedges, n);
}

// synthgen.hpp:76-85
Csr generate_erdos_renyi(int32_t n, double p, uint64_t seed) {
  if (n < 1) throw invalid_argument("n must be >= 1");
  if (p < 0.0 || p > 1.0) throw invalid_argument("p must be in [0, 1]");
  Mt64 rng(seed);
  std::vector<int32_t> e;
  for (int32_t u = 0; u < n; ++u)
    for (int32_t v = u + 1; v < n; ++v)
      if (rng.unit() < p) { e.push_back(u); e.push_back(v); }
  return csr_from_edges(e.data(), static_cast<int64_t>(e.size() / 2), n);
}

// ------------------------------------------------------------- color index
Binom::Binom() {
  std::memset(c, 0, sizeof(c));
  for (int a = 0; a <= kMaxK; ++a) {
    c[a][0] = 1;
    for (int b = 1; b <= a; ++b) c[a][b] = c[a - 1][b - 1] + (b <= a - 1 ? c[a - 1][b] : 0);
  }
}
const Binom& binom() { static const Binom b; return b; }

int64_t index_of(const int* colors, int h) {
  int64_t idx = 0;
  for (int pos = 1; pos <= h; ++pos) idx += binom()(colors[pos - 1], pos);
  return idx;
}

void set_of(int k, int64_t index, int h, int* colors) {
  int c = k - 1;
  for (int pos = h; pos >= 1; --pos) {
    while (binom()(c, pos) > index) --c;
    colors[pos - 1] = c;
    index -= binom()(c, pos);
    --c;
  }
}

uint32_t set_mask(int k, int64_t index, int h) {
  int cs[kMaxK];
  set_of(k, index, h, cs);
  uint32_t m = 0;
  for (int j = 0; j < h; ++j) m |= 1u << cs[j];
  return m;
}

// ------------------------------------------------- rooted-color compression
// Group assignment: start from g(S) = (sum of the colors of S) mod m, which is
// already balanced for most (k, s) (every color's sets spread evenly over the
// residues), then repair overfull (group, color) pairs by min-conflict moves.
// m starts at the lower bound ceil(C(k-1,s-1) / zw); a first-fit pass is the
// always-feasible fallback.  Deterministic (fixed-seed generator).
RootedLayout build_rooted_layout(int k, int s) {
  if (k < 1 || k > kMaxK || s < 1 || s > k) throw invalid_argument("rooted layout: bad (k, s)");
  const Binom& B = binom();
  RootedLayout L;
  L.k = k;
  L.s = s;
  const int64_t C = B(k, s), W = B(k - 1, s - 1);
  L.full_cols = static_cast<int32_t>(C);
  L.zw = W <= 8 ? 8 : (W <= 16 ? 16 : 32);
  const int zw = L.zw;
  std::vector<uint32_t> mask(static_cast<size_t>(C));
  std::vector<int> csum(static_cast<size_t>(C));
  int cs[kMaxK];
  for (int64_t x = 0; x < C; ++x) {
    set_of(k, x, s, cs);
    uint32_t m = 0;
    int sum = 0;
    for (int j = 0; j < s; ++j) { m |= 1u << cs[j]; sum += cs[j]; }
    mask[x] = m;
    csum[x] = sum;
  }
  std::vector<int> g(static_cast<size_t>(C));
  uint64_t rs = 0x9E3779B97F4A7C15ull;
  auto rnd = [&rs](uint64_t bound) {
    rs += 0x9E3779B97F4A7C15ull;
    uint64_t z = rs;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (z ^ (z >> 31)) % bound;
  };
  auto try_groups = [&](int m) -> bool {
    std::vector<int> cnt(static_cast<size_t>(m) * k, 0);
    std::vector<std::vector<int64_t>> members(static_cast<size_t>(m));
    std::vector<int64_t> where(static_cast<size_t>(C));
    for (int64_t x = 0; x < C; ++x) {
      const int gi = csum[x] % m;
      g[x] = gi;
      where[x] = static_cast<int64_t>(members[gi].size());
      members[gi].push_back(x);
      for (uint32_t b = mask[x]; b; b &= b - 1) ++cnt[static_cast<size_t>(gi) * k + __builtin_ctz(b)];
    }
    // overfull (group, color) pairs, kept as an indexable set
    std::vector<int> over, opos(static_cast<size_t>(m) * k, -1);
    auto sync = [&](int gi, int c) {
      const size_t id = static_cast<size_t>(gi) * k + c;
      const bool bad = cnt[id] > zw;
      if (bad && opos[id] < 0) { opos[id] = static_cast<int>(over.size()); over.push_back(static_cast<int>(id)); }
      if (!bad && opos[id] >= 0) {
        const int last = over.back();
        over[opos[id]] = last;
        opos[last] = opos[id];
        over.pop_back();
        opos[id] = -1;
      }
    };
    for (int gi = 0; gi < m; ++gi)
      for (int c = 0; c < k; ++c) sync(gi, c);
    const int64_t maxit = 4 * C + 20000;
    for (int64_t it = 0; it < maxit && !over.empty(); ++it) {
      const int id = over[rnd(over.size())];
      const int gi = id / k, c = id % k;
      auto& mem = members[gi];
      int64_t x = -1;
      for (int tries = 0; tries < 64 * k && x < 0; ++tries) {
        const int64_t y = mem[rnd(mem.size())];
        if (mask[y] >> c & 1u) x = y;
      }
      if (x < 0) continue;
      // best of (at most) 48 candidate groups
      int best = -1, bd = 1 << 30;
      const int ncand = std::min(m - 1, 48);
      for (int q = 0; q < ncand; ++q) {
        const int b = m - 1 <= 48 ? (q < gi ? q : q + 1) : static_cast<int>(rnd(m));
        if (b == gi) continue;
        int d = 0;
        for (uint32_t bb = mask[x]; bb; bb &= bb - 1) d += cnt[static_cast<size_t>(b) * k + __builtin_ctz(bb)] >= zw;
        if (d < bd || (d == bd && (rnd(4) == 0))) { bd = d; best = b; }
      }
      if (best < 0) return false;
      // move x: gi -> best
      const int64_t last = mem.back();
      mem[where[x]] = last;
      where[last] = where[x];
      mem.pop_back();
      where[x] = static_cast<int64_t>(members[best].size());
      members[best].push_back(x);
      g[x] = best;
      for (uint32_t bb = mask[x]; bb; bb &= bb - 1) {
        const int cc = __builtin_ctz(bb);
        --cnt[static_cast<size_t>(gi) * k + cc];
        ++cnt[static_cast<size_t>(best) * k + cc];
        sync(gi, cc);
        sync(best, cc);
      }
    }
    return over.empty();
  };
  const int lb = static_cast<int>((W + zw - 1) / zw);
  int m = -1;
  for (int step = 0; step < 6 && m < 0; ++step) {
    const int t = lb + (step == 0 ? 0 : (lb >> (6 - step)) + step);  // lb, +1/32, +1/16, ... +1/2
    if (try_groups(t)) m = t;
  }
  if (m < 0) {  // first fit in column order: always feasible
    std::vector<std::vector<int>> cnt;
    for (int64_t x = 0; x < C; ++x) {
      int gi = 0;
      for (;; ++gi) {
        if (gi == static_cast<int>(cnt.size())) cnt.emplace_back(k, 0);
        bool ok = true;
        for (uint32_t b = mask[x]; b && ok; b &= b - 1) ok = cnt[gi][__builtin_ctz(b)] < zw;
        if (ok) break;
      }
      g[x] = gi;
      for (uint32_t b = mask[x]; b; b &= b - 1) ++cnt[gi][__builtin_ctz(b)];
    }
    m = static_cast<int>(cnt.size());
  }
  // drop empty groups; members in ascending full-column order
  std::vector<std::vector<int64_t>> mem(static_cast<size_t>(m));
  for (int64_t x = 0; x < C; ++x) mem[g[x]].push_back(x);
  mem.erase(std::remove_if(mem.begin(), mem.end(), [](const std::vector<int64_t>& v) { return v.empty(); }),
            mem.end());
  L.groups = static_cast<int>(mem.size());
  L.perm.assign(static_cast<size_t>(C), -1);
  int32_t base = 0;
  for (int gi = 0; gi < L.groups; ++gi) {
    L.fbase.push_back(base);
    L.fsize.push_back(static_cast<int32_t>(mem[gi].size()));
    for (size_t a = 0; a < mem[gi].size(); ++a) L.perm[mem[gi][a]] = base + static_cast<int32_t>(a);
    base += (static_cast<int32_t>(mem[gi].size()) + 7) / 8 * 8;
  }
  L.store_cols = base;
  L.inv.assign(static_cast<size_t>(base), -1);
  for (int64_t x = 0; x < C; ++x) L.inv[L.perm[x]] = static_cast<int32_t>(x);
  const size_t slots = static_cast<size_t>(L.groups) * zw;
  L.slot_acc.assign(slots * k, -1);
  L.slot_col.assign(slots * k, -1);
  for (int c = 0; c < k; ++c)
    for (int gi = 0; gi < L.groups; ++gi) {
      int t = 0;
      for (size_t a = 0; a < mem[gi].size(); ++a) {
        const int64_t x = mem[gi][a];
        if (!(mask[x] >> c & 1u)) continue;
        if (t >= zw) throw logic_error("rooted layout: group over capacity");
        const size_t i = static_cast<size_t>(c) * slots + static_cast<size_t>(gi) * zw + t++;
        L.slot_acc[i] = static_cast<int16_t>(a);
        L.slot_col[i] = static_cast<int32_t>(x);
      }
    }
  return L;
}

SplitTable build_split_table(int k, int parent_size, int active_size) {
  const int passive_size = parent_size - active_size;
  if (active_size < 1 || passive_size < 1)
    throw invalid_argument("split requires nonempty active and passive children");
  if (parent_size > k) throw invalid_argument("sub-template larger than color count");
  const Binom& B = binom();
  SplitTable st;
  st.parent_size = parent_size;
  st.active_size = active_size;
  st.passive_size = passive_size;
  st.parent_cols = static_cast<int32_t>(B(k, parent_size));
  st.active_cols = static_cast<int32_t>(B(k, active_size));
  st.passive_cols = static_cast<int32_t>(B(k, passive_size));
  st.pairs_per_parent = static_cast<int>(B(parent_size, active_size));
  st.partners_per_passive = static_cast<int>(B(k - passive_size, active_size));
  const size_t total = static_cast<size_t>(st.parent_cols) * st.pairs_per_parent;
  st.active_index.resize(total);
  st.passive_index.resize(total);
  // Walk the active position subsets in lexicographic order as bitmasks
  // over the parent's sorted colors: next subset = Gosper-free odometer.
  std::vector<int> pos(active_size);
  int parent[kMaxK], act[kMaxK], pas[kMaxK];
  for (int32_t is = 0; is < st.parent_cols; ++is) {
    set_of(k, is, parent_size, parent);
    for (int j = 0; j < active_size; ++j) pos[j] = j;
    for (int p = 0; p < st.pairs_per_parent; ++p) {
      uint32_t chosen = 0;
      for (int j = 0; j < active_size; ++j) chosen |= 1u << pos[j];
      int na = 0, np = 0;
      for (int q = 0; q < parent_size; ++q) (chosen >> q & 1 ? act[na++] : pas[np++]) = parent[q];
      const size_t slot = static_cast<size_t>(is) * st.pairs_per_parent + p;
      st.active_index[slot] = static_cast<int32_t>(index_of(act, active_size));
      st.passive_index[slot] = static_cast<int32_t>(index_of(pas, passive_size));
      int j = active_size - 1;  // advance the odometer
      while (j >= 0 && pos[j] == parent_size - active_size + j) --j;
      if (j < 0) break;
      ++pos[j];
      for (int q = j + 1; q < active_size; ++q) pos[q] = pos[q - 1] + 1;
    }
  }
  // grouped view: bucket by passive column, order by (I_s, I_a)
  std::vector<int64_t> fill(static_cast<size_t>(st.passive_cols), 0);
  std::vector<std::pair<int32_t, int32_t>> grp(total);
  for (size_t s = 0; s < total; ++s) {
    const int32_t ip = st.passive_index[s];
    grp[static_cast<size_t>(ip) * st.partners_per_passive + fill[ip]++] = {
        static_cast<int32_t>(s / st.pairs_per_parent), st.active_index[s]};
  }
  st.grouped_parent.resize(total);
  st.grouped_active.resize(total);
  for (int32_t ip = 0; ip < st.passive_cols; ++ip) {
    if (fill[ip] != st.partners_per_passive) throw logic_error("split group size mismatch");
    auto* b = grp.data() + static_cast<size_t>(ip) * st.partners_per_passive;
    std::sort(b, b + st.partners_per_passive);
    for (int q = 0; q < st.partners_per_passive; ++q) {
      st.grouped_parent[static_cast<size_t>(ip) * st.partners_per_passive + q] = b[q].first;
      st.grouped_active[static_cast<size_t>(ip) * st.partners_per_passive + q] = b[q].second;
    }
  }
  return st;
}

// ---------------------------------------------------------------- template
static int lowest(uint32_t m) { return __builtin_ctz(m); }

// component of `from` inside `mask` without crossing into `blocked`
static uint32_t component(const Template& t, uint32_t mask, int from, int blocked) {
  uint32_t seen = 1u << from, frontier = seen;
  const uint32_t allowed = mask & ~(blocked >= 0 ? 1u << blocked : 0u);
  while (frontier) {
    uint32_t next = 0;
    for (uint32_t f = frontier; f; f &= f - 1) next |= t.adj[lowest(f)];
    next &= allowed & ~seen;
    seen |= next;
    frontier = next;
  }
  return seen;
}

Template make_template(int k, const int32_t* edges, int root) {
  if (k < 1) throw parse_error("not a tree: empty template");
  if (k > kMaxK) throw invalid_argument("color count k must be in [1, 20]");
  Template t;
  t.k = k;
  t.adj.assign(k, 0);
  int max_id = k == 1 ? 0 : -1;
  for (int e = 0; e < k - 1; ++e) {
    const int u = edges[2 * e], v = edges[2 * e + 1];
    if (u < 0 || v < 0 || u >= k || v >= k || u == v)
      throw parse_error("not a tree: bad edge " + std::to_string(u) + " " + std::to_string(v));
    max_id = std::max({max_id, u, v});
    t.edges.emplace_back(u, v);
    t.adj[u] |= 1u << v;
    t.adj[v] |= 1u << u;
  }
  if (max_id + 1 != k) throw parse_error("not a tree: vertex ids must be 0..k-1");
  const uint32_t all = k == 32 ? ~0u : (1u << k) - 1;
  if (component(t, all, 0, -1) != all) throw parse_error("not a tree: disconnected");
  if (root < 0) {  // templates.hpp:67-74: max degree, smallest id
    root = 0;
    for (int v = 1; v < k; ++v)
      if (__builtin_popcount(t.adj[v]) > __builtin_popcount(t.adj[root])) root = v;
  }
  if (root >= k) throw parse_error("template root out of range");
  t.root = root;
  return t;
}

// templates.hpp:180-210: node ids in pre-order, dp_order in post-order,
// active child (root side) built before the passive child (tau side).
static int build_plan(const Template& t, Plan& p, uint32_t mask, int root) {
  const int id = p.num_nodes++;
  p.size.push_back(__builtin_popcount(mask));
  p.node_root.push_back(root);
  p.active.push_back(-1);
  p.passive.push_back(-1);
  p.parent.push_back(-1);
  p.vertices.push_back(mask);
  if (p.size[id] > 1) {
    const int tau = lowest(t.adj[root] & mask);  // smallest-id neighbour inside
    const uint32_t act = component(t, mask, root, tau);
    const int a = build_plan(t, p, act, root);
    const int q = build_plan(t, p, mask & ~act, tau);
    p.active[id] = a;
    p.passive[id] = q;
    p.parent[a] = id;
    p.parent[q] = id;
  }
  p.dp_order.push_back(id);
  return id;
}

Plan partition(const Template& t) {
  Plan p;
  p.k = t.k;
  p.root = t.root;
  build_plan(t, p, t.k == 32 ? ~0u : (1u << t.k) - 1, t.root);
  return p;
}

// |Aut(T)| by bottom-up canonical class ids: two rooted subtrees get the same
// id iff isomorphic (ids interned from sorted child-id lists); the rooted
// automorphism count multiplies the children's counts and m! for every class
// appearing m times.  Anchored at the center(s) as templates.hpp:326-339.
namespace {
struct Canon {
  std::map<std::vector<int>, int> ids;
  const Template& t;
  explicit Canon(const Template& tt) : t(tt) {}
  std::pair<int, uint64_t> rooted(int v, int parent) {
    std::vector<int> kids;
    uint64_t aut = 1;
    for (uint32_t m = t.adj[v]; m; m &= m - 1) {
      const int w = lowest(m);
      if (w == parent) continue;
      auto [cid, caut] = rooted(w, v);
      kids.push_back(cid);
      aut *= caut;
    }
    std::sort(kids.begin(), kids.end());
    for (size_t i = 0; i < kids.size();) {
      size_t j = i;
      while (j < kids.size() && kids[j] == kids[i]) ++j;
      for (size_t r = 2; r <= j - i; ++r) aut *= r;
      i = j;
    }
    auto it = ids.emplace(std::move(kids), static_cast<int>(ids.size())).first;
    return {it->second, aut};
  }
};
}  // namespace

uint64_t automorphism_count(const Template& t) {
  if (t.k == 1) return 1;
  std::vector<int> deg(t.k);
  uint32_t alive = (1u << t.k) - 1, leaves = 0;
  for (int v = 0; v < t.k; ++v) {
    deg[v] = __builtin_popcount(t.adj[v]);
    if (deg[v] == 1) leaves |= 1u << v;
  }
  while (__builtin_popcount(alive) > 2) {  // peel leaves to the center(s)
    alive &= ~leaves;
    uint32_t next = 0;
    for (uint32_t m = leaves; m; m &= m - 1)
      for (uint32_t nb = t.adj[lowest(m)] & alive; nb; nb &= nb - 1)
        if (--deg[lowest(nb)] == 1) next |= 1u << lowest(nb);
    leaves = next;
  }
  Canon c(t);
  const int c0 = lowest(alive);
  if (__builtin_popcount(alive) == 1) return c.rooted(c0, -1).second;
  const int c1 = lowest(alive & (alive - 1));
  auto a = c.rooted(c0, c1);
  auto b = c.rooted(c1, c0);
  return a.second * b.second * (a.first == b.first ? 2 : 1);
}

int64_t estimate_bytes(const Plan& plan, int64_t n) {
  std::vector<char> live(plan.num_nodes, 0);
  int64_t peak = 0;
  for (int id : plan.dp_order) {
    live[id] = 1;
    int64_t cols = 0;
    for (int j = 0; j < plan.num_nodes; ++j)
      if (live[j]) cols += binom()(plan.k, plan.size[j]);
    peak = std::max(peak, cols);
    if (!plan.is_leaf(id)) live[plan.active[id]] = live[plan.passive[id]] = 0;
  }
  return 8 * n * peak;
}

double colorful_probability(int k) {
  double p = 1.0;
  for (int i = 1; i <= k; ++i) p *= static_cast<double>(i) / static_cast<double>(k);
  return p;
}

}  // namespace tcg
