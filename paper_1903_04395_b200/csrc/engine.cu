// engine.cu -- per-GPU DP engine (see engine.hpp).
#include "engine.hpp"
#include "kernels.cuh"
#include "kernels_rt.cuh"
#include "kernels_graph.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <type_traits>

namespace tcg {

#define TCG_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      if (e_ == cudaErrorMemoryAllocation) {                                              \
        cudaGetLastError();                                                               \
        throw resource_error(std::string("device allocation failed: ") + #call);          \
      }                                                                                   \
      throw cuda_error(std::string(cudaGetErrorString(e_)) + " at " + __FILE__ + ":" +   \
                       std::to_string(__LINE__));                                         \
    }                                                                                     \
  } while (0)

namespace {
// cudaFuncAttributeMaxDynamicSharedMemorySize is per (device, function), shared by every engine
// of the process: engines driven by different host threads (tcg_create_multi with a device listed
// twice, a batch engine next to its parent) launch the same kernel with different dynamic sizes,
// so the limit is only ever RAISED (a launch below the limit is always valid).
void smem_limit(const void* f, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  TCG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[{dev, f}];
  if (bytes > c) {
    TCG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    c = bytes;
  }
}

constexpr int64_t kAlign = 256;
int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

template <typename T>
T* dupload(const std::vector<T>& h, cudaStream_t s) {
  T* d = nullptr;
  TCG_CUDA(cudaMalloc(&d, sizeof(T) * std::max<size_t>(h.size(), 1)));
  if (!h.empty()) TCG_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s));
  return d;
}

// First-fit arena planner over the reference's liveness sequence.
struct ArenaPlanner {
  std::map<int64_t, int64_t> used;  // offset -> bytes
  int64_t peak = 0;
  int64_t alloc(int64_t bytes) {
    bytes = align_up(std::max<int64_t>(bytes, kAlign));
    int64_t off = 0;
    for (auto& [o, b] : used) {
      if (o - off >= bytes) break;
      off = std::max(off, o + b);
    }
    used[off] = bytes;
    refs[off] = 1;
    peak = std::max(peak, off + bytes);
    return off;
  }
  // a table shared by several consumers (deduplicated sub-templates) is
  // released by its last consumer
  std::map<int64_t, int> refs;
  void retain(int64_t off) { ++refs[off]; }
  void free(int64_t off) {
    if (--refs[off] <= 0) {
      used.erase(off);
      refs.erase(off);
    }
  }
};

// g(X2, i): combinadic contribution of the H2 colors of a set whose H1 part has
// i colors (they take positions 1..i) -- kernels.cuh ema_blocked.
int64_t h2_offset(uint32_t x2, int i) {
  int64_t off = 0;
  int pos = i;
  for (int c = 0; c < 32; ++c)
    if (x2 >> c & 1u) off += binom()(c, ++pos);
  return off;
}

// Output groups and blocks of the color-split eMA for a node (s, a) with k colors.
// h1: colors of the register-blocked H1 (pattern code i * shift + j)
void build_blocked(int k, int s, int a, std::vector<dev::GroupDesc>& groups,
                   std::vector<dev::BlockDesc>& blocks, int h1 = dev::kH1, int shift = 8) {
  const int p = s - a;
  struct G { dev::GroupDesc d; int64_t work; std::vector<dev::BlockDesc> b; };
  std::vector<G> gs;
  const uint32_t h2mask = (k >= 32 ? ~0u : ((1u << k) - 1)) & ~((1u << h1) - 1);
  int64_t total = 0;
  // all subsets S2 of H2
  for (uint32_t s2 = 0;; s2 = (s2 - h2mask) & h2mask) {
    const int t = __builtin_popcount(s2), s1 = s - t;
    if (s1 >= 0 && s1 <= h1) {
      G g;
      g.d = dev::GroupDesc{static_cast<int32_t>(h2_offset(s2, s1)), s1, 0, 0};
      g.work = 0;
      for (int i = std::max(0, s1 - p); i <= std::min(a, s1); ++i) {
        const int j = s1 - i, ac = a - i;
        if (ac < 0 || ac > t || p - j < 0) continue;
        // subsets a2 of s2 with |a2| = ac
        for (uint32_t a2 = 0;; a2 = (a2 - s2) & s2) {
          if (__builtin_popcount(a2) == ac) {
            const uint32_t p2 = s2 & ~a2;
            g.b.push_back(dev::BlockDesc{static_cast<int32_t>(h2_offset(a2, i)),
                                         static_cast<int32_t>(h2_offset(p2, j)), i * shift + j, 0});
            g.work += dev::cbin(h1, i) * dev::cbin(h1 - i, j);
          }
          if (a2 == s2) break;
        }
      }
      std::sort(g.b.begin(), g.b.end(), [](const dev::BlockDesc& x, const dev::BlockDesc& y) {
        return x.ij < y.ij || (x.ij == y.ij && x.a_off < y.a_off);
      });
      total += g.work;
      gs.push_back(std::move(g));
    }
    if (s2 == h2mask) break;
  }
  if (total != binom()(k, s) * binom()(s, a)) throw logic_error("blocked eMA does not cover every split pair");
  // (work descending; equal work: by s1, so the groups of one shape stay together)
  std::stable_sort(gs.begin(), gs.end(), [](const G& x, const G& y) {
    return x.work > y.work || (x.work == y.work && x.d.s1 < y.d.s1);
  });
  groups.clear();
  blocks.clear();
  for (auto& g : gs) {
    // pad of a run's first block = the run's length (runs of one (i, j) pattern)
    for (size_t b = 0; b < g.b.size();) {
      size_t e = b;
      while (e < g.b.size() && g.b[e].ij == g.b[b].ij) ++e;
      for (size_t q = b; q < e; ++q) g.b[q].pad = static_cast<int32_t>(q == b ? e - b : 0);
      b = e;
    }
    g.d.b0 = static_cast<int32_t>(blocks.size());
    blocks.insert(blocks.end(), g.b.begin(), g.b.end());
    g.d.b1 = static_cast<int32_t>(blocks.size());
    groups.push_back(g.d);
  }
}

// Tasks of the vertex-per-CTA blocked eMA (kernels_rt.cuh ema_rtv_blocked): the
// output groups of build_blocked, cut into tasks of gpt = 32 / V groups of one
// SHAPE (same s1 and the same sequence of pattern runs), so a warp walks one
// run list for all its lanes.  Descriptors {a_off | p_off << 16} are stored
// step-major per task (step q of group gl at blk0 + q * gpt + gl).  Inside a
// run any block order is valid; it is chosen (seeded multi-start greedy per
// step, then pairwise moves between steps) so that a step's A offsets (and P
// offsets) are equal -- one broadcast read -- or fall on distinct residues
// mod gpt, i.e. distinct shared-memory banks (the V vertices of a group sit
// 32 / V banks apart): 1.26x -> 1.12x the conflict-free wavefronts on cfg5
// node 1.  Padding lanes of a partial task repeat the
// first group's descriptor (a broadcast read) and have gout = -1.
struct RtvPlan {
  std::vector<dev::RtvTask> tasks;
  std::vector<int32_t> gout;
  std::vector<uint32_t> runs, blocks;
  int64_t steps = 0, wavefronts = 0, ideal = 0;  // (diagnostics: shared-load wavefronts per group pass vs conflict-free)
};
RtvPlan build_rtv_tasks(int k, int s, int a, int h1, int V) {
  std::vector<dev::GroupDesc> gr;
  std::vector<dev::BlockDesc> bl;
  build_blocked(k, s, a, gr, bl, h1, 16);
  const int gpt = 32 / V;
  RtvPlan P;
  uint32_t seed = 12345u;  // (fixed: the plan, and so the fp32 summation order, is reproducible)
  auto rnd = [&seed]() { return (seed = seed * 1664525u + 1013904223u) >> 8; };
  auto sig = [&](const dev::GroupDesc& g) {
    std::vector<uint32_t> r;
    for (int b = g.b0; b < g.b1; b += bl[b].pad)
      r.push_back(static_cast<uint32_t>(bl[b].ij) | (static_cast<uint32_t>(bl[b].pad) << 8));
    return r;
  };
  for (size_t gi = 0; gi < gr.size();) {
    const std::vector<uint32_t> rs = sig(gr[gi]);
    size_t ge = gi + 1;
    while (ge < gr.size() && gr[ge].s1 == gr[gi].s1 && sig(gr[ge]) == rs) ++ge;
    const int32_t run0 = static_cast<int32_t>(P.runs.size());
    for (uint32_t rr : rs)  // {i * 16 + j | len << 8} -> {hcode(i, j) | len << 8}
      P.runs.push_back(static_cast<uint32_t>(dev::hcode(static_cast<int>(rr & 0xFFu) / 16, static_cast<int>(rr & 0xFFu) % 16)) |
                       (rr & ~0xFFu));
    for (size_t c = gi; c < ge; c += gpt) {
      const int ng = static_cast<int>(std::min<size_t>(gpt, ge - c));
      P.tasks.push_back(dev::RtvTask{static_cast<int32_t>(P.blocks.size()), run0, static_cast<int32_t>(rs.size()),
                                     gr[gi].s1});
      for (int gl = 0; gl < gpt; ++gl) P.gout.push_back(gl < ng ? gr[c + gl].out_off : -1);
      int boff = 0;
      for (uint32_t rr : rs) {
        const int ij = static_cast<int>(rr & 0xFFu), len = static_cast<int>(rr >> 8);
        const int wa = dev::cbin(h1, ij / 16), wp = dev::cbin(h1, ij % 16);
        auto desc = [&](int gl, int b) -> const dev::BlockDesc& { return bl[gr[c + gl].b0 + boff + b]; };
        // shared-load wavefronts of a step: per operand, the largest number of DISTINCT offsets on
        // one residue (equal offsets are one broadcast read), weighted by the operand's loads
        auto step_cost = [&](const std::vector<int>& blk) {
          int ma = 0, mp = 0;
          for (int res = 0; res < gpt; ++res) {
            int ca = 0, cp = 0;
            int32_t sa[32], sp[32];
            for (int gl = 0; gl < ng; ++gl) {
              const dev::BlockDesc& d = desc(gl, blk[gl]);
              if (d.a_off % gpt == res && std::find(sa, sa + ca, d.a_off) == sa + ca) sa[ca++] = d.a_off;
              if (d.p_off % gpt == res && std::find(sp, sp + cp, d.p_off) == sp + cp) sp[cp++] = d.p_off;
            }
            ma = std::max(ma, ca);
            mp = std::max(mp, cp);
          }
          return ma * wa + mp * wp;
        };
        // 1. per step: greedy over the groups in several (seeded) orders, the cheapest kept
        std::vector<std::vector<char>> used(ng, std::vector<char>(len, 0));
        std::vector<std::vector<int>> assign(len, std::vector<int>(ng, 0));  // [step][group] -> block of the run
        std::vector<int> cost(len), order(ng), choice(ng);
        for (int q = 0; q < len; ++q) {
          int best_cost = 1 << 30;
          for (int trial = 0; trial < 16 && best_cost > wa + wp; ++trial) {
            for (int i = 0; i < ng; ++i) order[i] = i;
            if (trial)
              for (int i = ng - 1; i > 0; --i) std::swap(order[i], order[rnd() % (i + 1)]);
            int32_t ra[32], rp[32];
            for (int r = 0; r < gpt; ++r) ra[r] = rp[r] = -1;
            for (int oi = 0; oi < ng; ++oi) {
              const int gl = order[oi];
              int best = -1, bestc = 1 << 30;
              for (int b = 0; b < len && bestc > 0; ++b) {
                if (used[gl][b]) continue;
                const dev::BlockDesc& d = desc(gl, b);
                const int32_t xa = ra[d.a_off % gpt], xp = rp[d.p_off % gpt];
                const int cst = (xa >= 0 && xa != d.a_off ? wa : 0) + (xp >= 0 && xp != d.p_off ? wp : 0);
                if (cst < bestc) bestc = cst, best = b;
              }
              choice[gl] = best;
              ra[desc(gl, best).a_off % gpt] = desc(gl, best).a_off;
              rp[desc(gl, best).p_off % gpt] = desc(gl, best).p_off;
            }
            const int cst = step_cost(choice);
            if (cst < best_cost) best_cost = cst, assign[q] = choice;
          }
          cost[q] = best_cost;
          for (int gl = 0; gl < ng; ++gl) used[gl][assign[q][gl]] = 1;
        }
        // 2. local search: move one group's blocks between two steps while that lowers the cost
        for (int pass = 0; pass < 3; ++pass) {
          bool improved = false;
          for (int q1 = 0; q1 < len; ++q1) {
            if (cost[q1] == wa + wp) continue;
            for (int q2 = 0; q2 < len; ++q2) {
              if (q2 == q1) continue;
              for (int gl = 0; gl < ng; ++gl) {
                std::swap(assign[q1][gl], assign[q2][gl]);
                const int n1 = step_cost(assign[q1]), n2 = step_cost(assign[q2]);
                if (n1 + n2 < cost[q1] + cost[q2]) {
                  cost[q1] = n1, cost[q2] = n2, improved = true;
                } else {
                  std::swap(assign[q1][gl], assign[q2][gl]);
                }
              }
            }
          }
          if (!improved) break;
        }
        std::vector<uint32_t> pick(gpt);
        for (int q = 0; q < len; ++q) {
          for (int gl = 0; gl < ng; ++gl) {
            const dev::BlockDesc& d = desc(gl, assign[q][gl]);
            if (d.a_off >= 65536 || d.p_off >= 65536) throw logic_error("blocked eMA offsets exceed 16 bits");
            pick[gl] = static_cast<uint32_t>(d.a_off) | (static_cast<uint32_t>(d.p_off) << 16);
          }
          for (int gl = ng; gl < gpt; ++gl) pick[gl] = pick[0];
          P.blocks.insert(P.blocks.end(), pick.begin(), pick.end());
          ++P.steps;
          P.wavefronts += cost[q];
          P.ideal += wa + wp;
        }
        boff += len;
      }
    }
    gi = ge;
  }
  P.blocks.insert(P.blocks.end(), 128, 0u);  // (the kernel loads up to three 32-word chunks past a task)
  return P;
}

void release_schedule(PartSchedule& s) {
  if (!s.owned) {
    s = PartSchedule{};
    return;
  }
  dfree(s.d_segs);
  dfree(s.d_split_rows);
  dfree(s.d_slot_begin);
  dfree(s.d_slot_row);
  s = PartSchedule{};
}

// Cut row ranges [lo[v], hi[v]) into segments of <= kSegMax, counting-sort by
// length (descending), pad with no-op segments; rows longer than one segment
// get fp64 partial slots (summed in order by spmm_fixup).
PartSchedule build_schedule(const std::vector<int64_t>& lo, const std::vector<int64_t>& hi,
                            bool keep_empty, cudaStream_t stream) {
  const int32_t n = static_cast<int32_t>(lo.size());
  std::vector<dev::Seg> segs;
  segs.reserve(static_cast<size_t>(n) + 16);
  std::vector<int32_t> split_rows, slot_begin{0};
  int slot = 0;
  for (int32_t v = 0; v < n; ++v) {
    const int64_t d = hi[v] - lo[v];
    if (d == 0 && !keep_empty) continue;
    if (d <= dev::kSegMax) {
      segs.push_back({lo[v], static_cast<int32_t>(d), v});
    } else {
      split_rows.push_back(v);
      for (int64_t o = 0; o < d; o += dev::kSegMax)
        segs.push_back({lo[v] + o, static_cast<int32_t>(std::min<int64_t>(dev::kSegMax, d - o)), -1 - slot++});
      slot_begin.push_back(slot);
    }
  }
  std::vector<int64_t> pos(dev::kSegMax + 2, 0);
  for (auto& s : segs) pos[dev::kSegMax - s.len + 1]++;
  for (size_t i = 1; i < pos.size(); ++i) pos[i] += pos[i - 1];
  const int64_t padded = std::max<int64_t>((static_cast<int64_t>(segs.size()) + dev::kSegPad - 1) /
                                               dev::kSegPad * dev::kSegPad, dev::kSegPad);
  std::vector<dev::Seg> sorted(static_cast<size_t>(padded), dev::Seg{0, 0, dev::kSkip});
  for (auto& s : segs) sorted[pos[dev::kSegMax - s.len]++] = s;
  PartSchedule ps;
  ps.nseg_padded = padded;
  ps.d_segs = dupload(sorted, stream);
  ps.nsplit_rows = static_cast<int>(split_rows.size());
  ps.nslots = slot;
  if (ps.nsplit_rows) {
    ps.d_split_rows = dupload(split_rows, stream);
    ps.d_slot_begin = dupload(slot_begin, stream);
    std::vector<int32_t> slot_row(static_cast<size_t>(slot));
    for (int r = 0; r < ps.nsplit_rows; ++r)
      for (int q = slot_begin[r]; q < slot_begin[r + 1]; ++q) slot_row[q] = split_rows[r];
    ps.d_slot_row = dupload(slot_row, stream);
  }
  TCG_CUDA(cudaStreamSynchronize(stream));
  return ps;
}
}  // namespace

// Host-only self-check of the task layout of ema_rtv_blocked (tcg_rtv_task_layout): every
// (group, block) of build_blocked appears exactly once, in a task whose groups share one run
// list, at the descriptor position the kernel reads.  info = {tasks, groups, block steps, runs,
// shared-load wavefronts, conflict-free wavefronts}.
void rtv_task_layout_check(int k, int s, int a, int V, int64_t info[6]) {
  if (k < 2 || k > kMaxK || s < 2 || s > k || a < 1 || a >= s) throw invalid_argument("need 2 <= s <= k <= 20 and 1 <= a < s");
  if (V != 1 && V != 2 && V != 4 && V != 8) throw invalid_argument("V must be 1, 2, 4 or 8");
  if (k < dev::kH1) throw invalid_argument("need k >= 6 (the colours of the register-blocked part)");
  std::vector<dev::GroupDesc> gr;
  std::vector<dev::BlockDesc> bl;
  build_blocked(k, s, a, gr, bl, dev::kH1, 16);
  const RtvPlan P = build_rtv_tasks(k, s, a, dev::kH1, V);
  const int gpt = 32 / V;
  std::map<int32_t, size_t> by_out;
  for (size_t g = 0; g < gr.size(); ++g)
    if (!by_out.emplace(gr[g].out_off, g).second) throw logic_error("two groups share an output offset");
  std::vector<char> seen(gr.size(), 0);
  if (P.gout.size() != P.tasks.size() * static_cast<size_t>(gpt)) throw logic_error("gout size");
  for (size_t t = 0; t < P.tasks.size(); ++t) {
    const dev::RtvTask& task = P.tasks[t];
    for (int gl = 0; gl < gpt; ++gl) {
      const int32_t oo = P.gout[t * gpt + gl];
      if (oo < 0) continue;
      const auto it = by_out.find(oo);
      if (it == by_out.end() || seen[it->second]) throw logic_error("a task lists an unknown or repeated group");
      seen[it->second] = 1;
      const dev::GroupDesc& g = gr[it->second];
      if (g.s1 != task.s1) throw logic_error("task and group differ in s1");
      int64_t step = 0;
      int b = g.b0;
      for (int r = 0; r < task.nruns; ++r) {
        const uint32_t rr = P.runs[task.run0 + r];
        const int len = static_cast<int>(rr >> 8);
        std::vector<uint32_t> want, got;
        for (int q = 0; q < len; ++q, ++b, ++step) {
          if (b >= g.b1) throw logic_error("a task's runs are longer than its group's block list");
          if (static_cast<uint32_t>(dev::hcode(bl[b].ij / 16, bl[b].ij % 16)) != (rr & 0xFFu)) throw logic_error("run pattern differs from the group's blocks");
          want.push_back(static_cast<uint32_t>(bl[b].a_off) | (static_cast<uint32_t>(bl[b].p_off) << 16));
          got.push_back(P.blocks[task.blk0 + step * gpt + gl]);
        }
        std::sort(want.begin(), want.end());
        std::sort(got.begin(), got.end());
        if (want != got) throw logic_error("a run's descriptors are not a permutation of the group's blocks");
      }
      if (b != g.b1) throw logic_error("a task's runs do not cover its group's block list");
    }
  }
  for (char c : seen)
    if (!c) throw logic_error("a group is in no task");
  info[0] = static_cast<int64_t>(P.tasks.size());
  info[1] = static_cast<int64_t>(gr.size());
  info[2] = P.steps;
  info[3] = static_cast<int64_t>(P.runs.size());
  info[4] = P.wavefronts;
  info[5] = P.ideal;
}

Engine::Engine(const tcg_config& cfg, cudaStream_t shared_stream) : cfg_(cfg) {
  int ndev = 0;
  TCG_CUDA(cudaGetDeviceCount(&ndev));
  if (cfg.device < 0 || cfg.device >= ndev)
    throw invalid_argument("CUDA device " + std::to_string(cfg.device) + " not present (" +
                           std::to_string(ndev) + " visible)");
  TCG_CUDA(cudaSetDevice(cfg.device));
  cudaDeviceProp prop;
  TCG_CUDA(cudaGetDeviceProperties(&prop, cfg.device));
  num_sms_ = prop.multiProcessorCount;
  if (prop.major != 10)
    throw cuda_error("treecount-b200 is built for sm_100a (B200); device is sm_" +
                     std::to_string(prop.major) + std::to_string(prop.minor));
  if (const char* e = std::getenv("TCG_PART_KB")) part_bytes_ = std::max(1ll, std::atoll(e)) << 10;  // tests
  // rooted SpMM: ONE part (whole rows, one launch per group) unless
  // TCG_ROOTED_PARTS=1 splits it into colour classes of ~part_bytes_.  Every
  // extra part re-reads and re-writes the group's P' columns; measured on
  // B200 that costs more than the L2 misses of the unsplit gather source
  // (cfg3 49.9 -> 47.9 ms, cfg4 1666 -> 1049 ms).
  if (const char* e = std::getenv("TCG_ROOTED_PARTS")) rooted_part_mb_ = std::atoi(e);
  if (shared_stream) {
    stream_ = shared_stream;
    own_stream_ = false;
  } else {
    TCG_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  }
  TCG_CUDA(cudaMalloc(&d_scalars_, 64));
  TCG_CUDA(cudaMalloc(&d_seeds_, 1024 * sizeof(uint64_t)));
}

Engine::~Engine() {
  cudaSetDevice(cfg_.device);
  release_template();
  release_graph();
  free_graph_buffers();
  dfree(d_scalars_);
  dfree(d_seeds_);
  dfree(d_colors_);
  if (next_.stream) cudaStreamSynchronize(next_.stream);
  dfree(next_.d_buf[0]);
  dfree(next_.d_buf[1]);
  dfree(next_.d_seed);
  if (next_.ready) cudaEventDestroy(next_.ready);
  if (next_.stream) cudaStreamDestroy(next_.stream);
  batches_.clear();
  tr_.reset();  // (a communicator before its streams)
  if (comm_) cudaStreamDestroy(comm_);
  for (cudaEvent_t e : {ev_in_, ev_g_[0], ev_g_[1], ev_u_[0], ev_u_[1]})
    if (e) cudaEventDestroy(e);
  if (stream_ && own_stream_) cudaStreamDestroy(stream_);
}

void Engine::ensure_comm() {
  if (comm_) return;
  TCG_CUDA(cudaStreamCreateWithFlags(&comm_, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&ev_in_, &ev_g_[0], &ev_g_[1], &ev_u_[0], &ev_u_[1]})
    TCG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

void Engine::free_graph_buffers() {
  dfree(d_row_ptr_);
  dfree(d_col_);
  dfree(d_est_acc_);
  dfree(d_est_tot_);
  row_ptr_cap_ = col_cap_ = est_acc_cap_ = est_tot_cap_ = 0;
  dfree(gp_buf_);
  gp_n_cap_ = gp_nnz_cap_ = -1;
  dfree(gp_tmp_);
  gp_tmp_cap_ = 0;
  dfree(d_tile_tot_);
  tile_tot_cap_ = 0;
  dfree(d_counter_);
  dfree(d_perm_);
  dfree(d_inv_);
  perm_cap_ = inv_cap_ = 0;
  dfree(d_rp2_);
  dfree(d_col2_);
  rp2_cap_ = col2_cap_ = 0;
  dfree(rl_buf_);
  rl_cap_ = -1;
  dfree(d_colors_rl_);
  colors_rl_cap_ = 0;
  dfree(d_pv_out_);
  pv_out_cap_ = 0;
  dfree(d_urp_);
  dfree(d_ucol_);
  urp_cap_ = ucol_cap_ = 0;
}

void Engine::release_graph() {  // (d_row_ptr_ / d_col_ stay allocated for the next graph)
  for (auto& kv : sched_)
    for (auto& s : kv.second) release_schedule(s);
  sched_.clear();
  d_row_order_ = nullptr;  // (graph-prep block; d_tile_tot_ / d_counter_ are kept)
  dfree(d_xfull_);
  dfree(d_xfull2_);
  dfree(d_colors_pad_);
  dfree(d_gather_);
  dfree(d_rows_);
  d_lchunks_ = nullptr;
  d_lfirst_ = nullptr;
  nlchunks_ = 0;
  host_row_ptr_.clear();
  host_col_.clear();
  host_col_.shrink_to_fit();
  relabeled_ = false;
  rows_sorted_ = true;
  n_ = -1;
}

void Engine::release_template() {
  for (auto& e : exec_) {
    dfree(e.d_split);
    dfree(e.d_drop);
    dfree(e.d_packed);
    dfree(e.d_groups);
    dfree(e.d_blocks);
    dfree(e.d_slot_acc);
    dfree(e.d_slot_col);
    dfree(e.d_pinv);
    dfree(e.d_xmap);
    dfree(e.d_xmap_v);
    dfree(e.d_pmap);
    dfree(e.d_cmap);
    dfree(e.d_imap);
    dfree(e.d_omap);
    dfree(e.d_rt_packed);
    dfree(e.d_rt_split);
    dfree(e.d_rt_groups);
    dfree(e.d_rt_blocks);
    dfree(e.d_rtv_blocks);
    dfree(e.d_rtv_tasks);
    dfree(e.d_rtv_gout);
    dfree(e.d_rtv_runs);
    dfree(e.d_rtv_drop);
    dfree(e.d_emap);
    dfree(e.d_amap);
  }
  exec_.clear();
  dfree(arena_);
  arena_alloc_ = 0;
  dfree(d_partial_);
  partial_bytes_ = partial_alloc_ = 0;
  have_template_ = false;
  tables_valid_ = false;
}

// ------------------------------------------------------------------ graph
void Engine::set_shard(int rank, int world, std::unique_ptr<Transport> t) {
  if (world < 1 || rank < 0 || rank >= world) throw invalid_argument("bad shard rank/world");
  if (n_ >= 0) throw invalid_argument("tcg_set_shard_* must be called before tcg_set_graph");
  rank_ = rank;
  world_ = world;
  tr_ = std::move(t);
  if (have_template_) {  // layouts depend on sharding (no pair layout): re-plan the template
    std::vector<int32_t> edges;
    for (const auto& pr : tpl_.edges) {
      edges.push_back(pr.first);
      edges.push_back(pr.second);
    }
    set_template(tpl_.k, edges.data(), tpl_.root);
  }
}

void Engine::set_graph(const Csr& gin) {
  if (!sharded()) {
    set_graph_ptrs(gin.n, gin.row_ptr.data(), gin.col.data(), false);
    return;
  }
  TCG_CUDA(cudaSetDevice(cfg_.device));
  release_graph();
  Csr local;
  const Csr* gp = &gin;
  nglob_ = gin.n;
  if (sharded()) {
    // this rank's rows, padded to the largest shard; neighbour ids remapped
    // to padded-global (rank * nmax + local row) so the all-gathered panel is
    // indexed directly
    rows_ = shard_bounds(gin.n, gin.row_ptr.data(), world_);
    int64_t nmax = 1;
    for (int r = 0; r < world_; ++r) nmax = std::max(nmax, rows_[r + 1] - rows_[r]);
    nloc_ = static_cast<int32_t>(rows_[rank_ + 1] - rows_[rank_]);
    local.n = static_cast<int32_t>(nmax);
    local.row_ptr.assign(static_cast<size_t>(nmax) + 1, 0);
    const int64_t r0 = rows_[rank_];
    for (int32_t i = 0; i < nmax; ++i)
      local.row_ptr[i + 1] = local.row_ptr[i] + (i < nloc_ ? gin.row_ptr[r0 + i + 1] - gin.row_ptr[r0 + i] : 0);
    local.col.resize(static_cast<size_t>(local.row_ptr[nmax]));
    const int64_t e0 = gin.row_ptr[r0];
    parallel_for(local.row_ptr[nmax], [&](int64_t b, int64_t e1, int) {
      for (int64_t e = b; e < e1; ++e) {
        const int32_t u = gin.col[e0 + e];
        const int r = static_cast<int>(std::upper_bound(rows_.begin(), rows_.end(), static_cast<int64_t>(u)) - rows_.begin()) - 1;
        local.col[e] = static_cast<int32_t>(r * nmax + (u - rows_[r]));
      }
    });
    gp = &local;
    nsrc_ = static_cast<int32_t>(world_ * nmax);
    if (static_cast<int64_t>(world_) * nmax > INT32_MAX) throw invalid_argument("sharded graph too large");
  } else {
    rows_ = {0, static_cast<int64_t>(gin.n)};
    nloc_ = gin.n;
    nsrc_ = gin.n;
  }
  const Csr& g = *gp;
  n_ = g.n;
  nnz_ = g.nnz();
  TCG_CUDA(cudaMalloc(&d_xfull_, sizeof(float) * dev::kZ * std::max<int64_t>(nsrc_, 1)));
  if (tr_ && tr_->async()) {  // double buffer + communication stream (rooted_spmm prefetch)
    TCG_CUDA(cudaMalloc(&d_xfull2_, sizeof(float) * dev::kZ * std::max<int64_t>(nsrc_, 1)));
    ensure_comm();
  }
  TCG_CUDA(cudaMalloc(&d_colors_pad_, std::max<int64_t>(nsrc_, 1)));
  // [0, 2048): this rank's totals chunk; [2048, 2048 * (world + 1)): gathered
  TCG_CUDA(cudaMalloc(&d_gather_, sizeof(double) * 2048 * (world_ + 1)));
  d_rows_ = dupload(rows_, stream_);
  host_col_ = g.col;  // (the sharded CSR is a local copy anyway)
  finish_graph(g.row_ptr.data(), g.col.data(), false);
}

// Unsharded graph straight from caller buffers (not copied on the host): the
// CSR goes host -> device once (pinned buffers make this a full-speed DMA),
// is validated on the device when `validate`, and only O(n) host work builds
// the whole-row schedule and the degree order.  Vertex-range part schedules
// (full-table SpMM only) are built on first use (ensure_schedules).
void Engine::set_graph_ptrs(int32_t n, const int64_t* row_ptr, const int32_t* col, bool validate, int64_t nnz) {
  TCG_CUDA(cudaSetDevice(cfg_.device));
  release_graph();
  nglob_ = n;
  rows_ = {0, static_cast<int64_t>(n)};
  nloc_ = n;
  nsrc_ = n;
  n_ = n;
  nnz_ = nnz >= 0 ? nnz : row_ptr[n];  // (nnz given: device buffers, e.g. a batch union)
  finish_graph(row_ptr, col, validate);
}

// graph.hpp:65-95 from_edges ON THE DEVICE (kernels_graph.cuh edges_*): the
// caller's raw edge list (possibly directed, duplicated, self-looped) -> the
// reference's CSR (symmetric union, no loops, no duplicates, rows ascending)
// built in d_row_ptr_ / d_col_ by one radix sort, then the usual
// relabeling and schedules.  n_hint < 0: max id + 1.
void Engine::set_graph_edges(const int32_t* edges, int64_t m, int32_t n_hint) {
  if (sharded()) throw invalid_argument("tcg_set_graph_edges is not available on a sharded context");
  if (m < 0) throw invalid_argument("negative edge count");
  if (m > (int64_t{1} << 29)) throw invalid_argument("edge list too long for the device CSR build (2^29 edges)");
  TCG_CUDA(cudaSetDevice(cfg_.device));
  release_graph();
  const int64_t cnt = 2 * m;
  int32_t* dE = nullptr;
  uint64_t *k1 = nullptr, *k2 = nullptr;
  int32_t *keep = nullptr, *pos = nullptr;
  int64_t* deg = nullptr;
  auto cleanup = [&] {
    dfree(dE); dfree(k1); dfree(k2); dfree(keep); dfree(pos); dfree(deg);
  };
  try {
    TCG_CUDA(cudaMalloc(&dE, sizeof(int32_t) * std::max<int64_t>(cnt, 2) + 16));
    int32_t* mm = dE + std::max<int64_t>(cnt, 2);  // {max, min}
    const int32_t init[2] = {INT32_MIN, INT32_MAX};
    TCG_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, stream_));
    if (cnt) {
      TCG_CUDA(cudaMemcpyAsync(dE, edges, sizeof(int32_t) * cnt, cudaMemcpyDefault, stream_));
      dev::edges_minmax<<<148 * 4, 256, 0, stream_>>>(dE, cnt, mm, mm + 1);
    }
    int32_t h[2];
    copy_sync(h, mm, sizeof(h), cudaMemcpyDeviceToHost);
    const int32_t n = n_hint >= 0 ? n_hint : (cnt ? h[0] + 1 : 0);
    if (cnt && (h[1] < 0 || h[0] >= n)) throw parse_error("vertex id out of range [0, " + std::to_string(n) + ")");
    int bits = 1;
    while ((int64_t{1} << bits) < n) ++bits;
    TCG_CUDA(cudaMalloc(&deg, sizeof(int64_t) * (static_cast<size_t>(n) + 1)));
    TCG_CUDA(cudaMemsetAsync(deg, 0, sizeof(int64_t) * (static_cast<size_t>(n) + 1), stream_));
    int64_t nnz = 0;
    if (cnt) {
      TCG_CUDA(cudaMalloc(&k1, sizeof(uint64_t) * cnt));
      TCG_CUDA(cudaMalloc(&k2, sizeof(uint64_t) * cnt));
      TCG_CUDA(cudaMalloc(&keep, sizeof(int32_t) * cnt));
      TCG_CUDA(cudaMalloc(&pos, sizeof(int32_t) * cnt));
      dev::edges_keys<<<148 * 8, 256, 0, stream_>>>(dE, m, bits, k1);
      size_t b = 0;
      TCG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b, k1, k2, static_cast<int>(cnt), 0, 2 * bits, stream_));
      TCG_CUDA(cub::DeviceRadixSort::SortKeys(cub_tmp(b), b, k1, k2, static_cast<int>(cnt), 0, 2 * bits, stream_));
      dev::edges_keep<<<148 * 8, 256, 0, stream_>>>(k2, cnt, bits, keep, deg);
      b = 0;
      TCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, keep, pos, static_cast<int>(cnt), stream_));
      TCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp(b), b, keep, pos, static_cast<int>(cnt), stream_));
      int32_t tail[2];
      TCG_CUDA(cudaMemcpyAsync(&tail[0], pos + cnt - 1, 4, cudaMemcpyDeviceToHost, stream_));
      TCG_CUDA(cudaMemcpyAsync(&tail[1], keep + cnt - 1, 4, cudaMemcpyDeviceToHost, stream_));
      TCG_CUDA(cudaStreamSynchronize(stream_));
      nnz = static_cast<int64_t>(tail[0]) + tail[1];
    }
    if (row_ptr_cap_ < static_cast<int64_t>(n) + 1) {
      dfree(d_row_ptr_);
      row_ptr_cap_ = 0;
      TCG_CUDA(cudaMalloc(&d_row_ptr_, sizeof(int64_t) * (static_cast<size_t>(n) + 1)));
      row_ptr_cap_ = static_cast<int64_t>(n) + 1;
    }
    if (col_cap_ < std::max<int64_t>(nnz, 1)) {
      dfree(d_col_);
      col_cap_ = 0;
      TCG_CUDA(cudaMalloc(&d_col_, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
      col_cap_ = std::max<int64_t>(nnz, 1);
    }
    size_t b = 0;
    TCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, deg, d_row_ptr_, n + 1, stream_));
    TCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp(b), b, deg, d_row_ptr_, n + 1, stream_));
    if (cnt) dev::edges_emit<<<148 * 8, 256, 0, stream_>>>(k2, keep, pos, cnt, bits, d_col_);
    TCG_CUDA(cudaGetLastError());
    TCG_CUDA(cudaStreamSynchronize(stream_));
    nglob_ = n;
    rows_ = {0, static_cast<int64_t>(n)};
    nloc_ = n;
    nsrc_ = n;
    n_ = n;
    nnz_ = nnz;
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  finish_graph(nullptr, nullptr, false);
}

// CSR of the caller's vertices (the relabeling undone): row_ptr[n+1], col[nnz]
// (nullable), rows ascending -- inspection of a device-built graph.
void Engine::graph_csr(int32_t* n_out, int64_t* nnz_out, int64_t* row_ptr, int32_t* col) {
  if (n_ < 0) throw invalid_argument("no graph set (tcg_set_graph)");
  if (sharded()) throw invalid_argument("graph CSR is not inspectable on a sharded context");
  if (n_out) *n_out = nglob_;
  if (nnz_out) *nnz_out = nnz_;
  if (!row_ptr && !col) return;
  std::vector<int64_t> rp(static_cast<size_t>(n_) + 1);
  std::vector<int32_t> cl(static_cast<size_t>(std::max<int64_t>(nnz_, 1)));
  copy_sync(rp.data(), d_row_ptr_, sizeof(int64_t) * rp.size(), cudaMemcpyDeviceToHost);
  if (nnz_) copy_sync(cl.data(), d_col_, sizeof(int32_t) * nnz_, cudaMemcpyDeviceToHost);
  const std::vector<int32_t> perm = host_perm();
  std::vector<int64_t> deg(static_cast<size_t>(nglob_) + 1, 0);
  for (int32_t i = 0; i < n_; ++i) deg[perm[i]] = rp[i + 1] - rp[i];
  std::vector<int64_t> out_rp(static_cast<size_t>(nglob_) + 1, 0);
  for (int32_t v = 0; v < nglob_; ++v) out_rp[v + 1] = out_rp[v] + deg[v];
  if (row_ptr) std::copy(out_rp.begin(), out_rp.end(), row_ptr);
  if (col)
    for (int32_t i = 0; i < n_; ++i) {
      int32_t* dst = col + out_rp[perm[i]];
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) *dst++ = perm[cl[e]];
      std::sort(col + out_rp[perm[i]], dst);
    }
}

void Engine::finish_graph(const int64_t* row_ptr, const int32_t* col, bool validate) {
  static const bool timing = std::getenv("TCG_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  host_row_ptr_.clear();  // (host copy made lazily by ensure_schedules)
  if (row_ptr_cap_ < n_ + 1) {
    dfree(d_row_ptr_);
    row_ptr_cap_ = 0;
    TCG_CUDA(cudaMalloc(&d_row_ptr_, sizeof(int64_t) * (n_ + 1)));
    row_ptr_cap_ = n_ + 1;
  }
  if (col_cap_ < std::max<int64_t>(nnz_, 1)) {
    dfree(d_col_);
    col_cap_ = 0;
    TCG_CUDA(cudaMalloc(&d_col_, sizeof(int32_t) * std::max<int64_t>(nnz_, 1)));
    col_cap_ = std::max<int64_t>(nnz_, 1);
  }
  // (cudaMemcpyDefault: host buffers from the caller, device buffers from a
  // batch union; row_ptr == nullptr: the CSR was built in place, set_graph_edges)
  if (row_ptr) {
    TCG_CUDA(cudaMemcpyAsync(d_row_ptr_, row_ptr, sizeof(int64_t) * (n_ + 1), cudaMemcpyDefault, stream_));
    if (nnz_) TCG_CUDA(cudaMemcpyAsync(d_col_, col, sizeof(int32_t) * nnz_, cudaMemcpyDefault, stream_));
  }
  if (validate && nnz_) {
    TCG_CUDA(cudaMemsetAsync(reinterpret_cast<int*>(d_scalars_ + 4), 0, sizeof(int), stream_));
    dev::validate_csr<<<148 * 8, 256, 0, stream_>>>(d_row_ptr_, d_col_, n_, reinterpret_cast<int*>(d_scalars_ + 4));
    ++launches_;
  }
  if (validate && nnz_) {  // (before the relabeling reads the ids)
    int bad = 0;
    copy_sync(&bad, reinterpret_cast<int*>(d_scalars_ + 4), sizeof(int), cudaMemcpyDeviceToHost);
    if (bad) {
      const int32_t n = n_;
      release_graph();
      if (bad == 1) throw parse_error("CSR column out of range [0, " + std::to_string(n) + ") or self-loop");
      throw parse_error("CSR row not strictly ascending");
    }
  }
  static const int relabel_mode = [] {
    const char* s = std::getenv("TCG_RELABEL");
    return s ? std::atoi(s) : 1;
  }();
  if (relabel_mode && !no_relabel_ && !sharded() && n_ > 0) relabel_device();
  ++graph_gen_;
  if (timing) TCG_CUDA(cudaStreamSynchronize(stream_));
  const auto t1 = now();
  // Part size: dense rows (cfg3, avg degree ~200) gain from 64 MB parts; on
  // sparse skewed graphs (cfg2, avg ~30) the hub rows stay L2-resident anyway
  // and extra parts only add output passes (measured: profiles/ DESIGN.md 3).
  if (!std::getenv("TCG_PART_KB"))
    part_bytes_ = (n_ > 0 && nnz_ / std::max(n_, 1) >= 64) ? (64ll << 20) : (128ll << 20);
  max_slots_ = 0;
  const auto t2 = now();
  prep_graph_device();  // whole-row schedule, degree order, hub chunks (kernels_graph.cuh)
  max_slots_ = sched_[1][0].nslots;
  if (!d_counter_) TCG_CUDA(cudaMalloc(&d_counter_, 64));
  const auto t3 = now();
  const int64_t ntiles = (n_ + dev::kTileV - 1) / dev::kTileV;
  ensure_tile_tot(std::max<int64_t>(ntiles, static_cast<int64_t>(batch_copies_) * dev::kRootChunks));
  TCG_CUDA(cudaStreamSynchronize(stream_));
  const auto t4 = now();
  if (have_template_) plan_arena();
  if (timing)
    std::fprintf(stderr, "[tcg timing] set_graph: h2d+validate %.1f, device prep %.1f, sync %.1f, plan %.1f ms\n",
                 ms(t0, t1), ms(t2, t3), ms(t3, t4), ms(t4, now()));
  tables_valid_ = false;
}

void* Engine::cub_tmp(size_t need) {
  if (need > gp_tmp_cap_) {
    dfree(gp_tmp_);
    gp_tmp_cap_ = 0;
    TCG_CUDA(cudaMalloc(&gp_tmp_, need));
    gp_tmp_cap_ = need;
  }
  return gp_tmp_;
}

// Degree-aware relabeling with isolated-vertex compaction, on the device
// (kernels_graph.cuh relabel_*): the CSR in d_row_ptr_ / d_col_ is replaced
// by the CSR of the live vertices in descending-degree order, each row's new
// ids sorted ascending (a segmented sort), so the graph invariants hold for
// the schedules built next.  Counts of the caller's vertex v are those of
// internal row inv[v]; isolated vertices count 0 for every k >= 2.
void Engine::relabel_device() {
  const int64_t n = n_, nnz = nnz_;
  auto grow = [&](auto*& p, int64_t& cap, int64_t need, size_t elem) {
    if (cap >= need) return;
    dfree(p);
    cap = 0;
    TCG_CUDA(cudaMalloc(&p, elem * static_cast<size_t>(std::max<int64_t>(need, 1))));
    cap = need;
  };
  grow(d_perm_, perm_cap_, n, sizeof(int32_t));
  grow(d_inv_, inv_cap_, n, sizeof(int32_t));
  grow(d_rp2_, rp2_cap_, n + 1, sizeof(int64_t));
  grow(d_col2_, col2_cap_, nnz, sizeof(int32_t));
  const int64_t o_key = 0, o_key2 = (4 * n + 255) / 256 * 256, o_ids = 2 * o_key2, o_deg = 3 * o_key2,
                o_cnt = o_deg + (8 * (n + 1) + 255) / 256 * 256, need = o_cnt + 256;
  if (need > rl_cap_) {
    dfree(rl_buf_);
    rl_cap_ = -1;
    TCG_CUDA(cudaMalloc(&rl_buf_, need));
    rl_cap_ = need;
  }
  uint32_t* key = reinterpret_cast<uint32_t*>(rl_buf_ + o_key);
  uint32_t* key2 = reinterpret_cast<uint32_t*>(rl_buf_ + o_key2);
  int32_t* ids = reinterpret_cast<int32_t*>(rl_buf_ + o_ids);
  int64_t* deg = reinterpret_cast<int64_t*>(rl_buf_ + o_deg);
  int32_t* cnt = reinterpret_cast<int32_t*>(rl_buf_ + o_cnt);
  TCG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t), stream_));
  const unsigned g1 = static_cast<unsigned>((n + 255) / 256);
  dev::relabel_keys<<<g1, 256, 0, stream_>>>(d_row_ptr_, n_, key, ids, cnt);
  size_t b = 0;
  TCG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, key, key2, ids, d_perm_, static_cast<int>(n), 0, 32, stream_));
  TCG_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp(b), b, key, key2, ids, d_perm_, static_cast<int>(n), 0, 32, stream_));
  int32_t nact = 0;
  copy_sync(&nact, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost);
  TCG_CUDA(cudaMemsetAsync(d_inv_, 0xFF, sizeof(int32_t) * n, stream_));
  dev::relabel_inverse<<<static_cast<unsigned>((nact + 1 + 255) / 256), 256, 0, stream_>>>(d_row_ptr_, d_perm_, nact, d_inv_, deg);
  b = 0;
  TCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, deg, d_rp2_, static_cast<int>(nact + 1), stream_));
  TCG_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp(b), b, deg, d_rp2_, static_cast<int>(nact + 1), stream_));
  if (nnz > 0) {
    dev::relabel_fill<<<148 * 8, 256, 0, stream_>>>(d_row_ptr_, d_col_, d_perm_, d_inv_, d_rp2_, nact, d_col2_);
    std::swap(d_col_, d_col2_);
    std::swap(col_cap_, col2_cap_);
  }
  std::swap(d_row_ptr_, d_rp2_);
  std::swap(row_ptr_cap_, rp2_cap_);
  // (a row's new ids are in the order of its old ids: only the vertex-range
  // part schedules of the full-table SpMM need ascending rows -- sort_rows)
  rows_sorted_ = nnz == 0;
  TCG_CUDA(cudaGetLastError());
  n_ = nact;
  nsrc_ = nact;
  relabeled_ = true;
}

// Rows ascending (the vertex-range parts of the full-table SpMM cut rows by
// id): a segmented sort of the relabeled rows, on first need.
void Engine::sort_rows() {
  if (rows_sorted_) return;
  size_t b = 0;
  TCG_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, b, d_col_, d_col2_, static_cast<int>(nnz_), n_, d_row_ptr_,
                                              d_row_ptr_ + 1, stream_));
  TCG_CUDA(cub::DeviceSegmentedSort::SortKeys(cub_tmp(b), b, d_col_, d_col2_, static_cast<int>(nnz_), n_, d_row_ptr_,
                                              d_row_ptr_ + 1, stream_));
  std::swap(d_col_, d_col2_);
  std::swap(col_cap_, col2_cap_);
  TCG_CUDA(cudaStreamSynchronize(stream_));
  host_col_.clear();
  rows_sorted_ = true;
}

std::vector<int32_t> Engine::host_perm() {
  std::vector<int32_t> p(static_cast<size_t>(std::max(n_, 0)));
  if (relabeled_ && n_ > 0) copy_sync(p.data(), d_perm_, sizeof(int32_t) * n_, cudaMemcpyDeviceToHost);
  else for (int32_t i = 0; i < n_; ++i) p[i] = i;
  return p;
}

// per-vertex fp64 values of the internal rows -> caller order (host), 0 for
// isolated vertices; enqueued on stream_ (the caller synchronizes)
void Engine::unpermute_to_host(const double* d_internal, double* host) {
  if (!relabeled_) {
    TCG_CUDA(cudaMemcpyAsync(host, d_internal, sizeof(double) * n_, cudaMemcpyDeviceToHost, stream_));
    return;
  }
  if (pv_out_cap_ < nglob_) {
    dfree(d_pv_out_);
    pv_out_cap_ = 0;
    TCG_CUDA(cudaMalloc(&d_pv_out_, sizeof(double) * std::max<int64_t>(nglob_, 1)));
    pv_out_cap_ = nglob_;
  }
  TCG_CUDA(cudaMemsetAsync(d_pv_out_, 0, sizeof(double) * nglob_, stream_));
  if (n_ > 0)
    dev::scatter_rows_f64<<<static_cast<unsigned>((n_ + 255) / 256), 256, 0, stream_>>>(d_internal, d_perm_, n_, d_pv_out_);
  TCG_CUDA(cudaMemcpyAsync(host, d_pv_out_, sizeof(double) * nglob_, cudaMemcpyDeviceToHost, stream_));
}

// Whole-row segment schedule (sched_[1]), degree order and hub-row chunks of
// the bucketing, built on the device from d_row_ptr_ (same result as the
// host builders; kernels_graph.cuh).  Buffers are carved from one block kept
// across graphs that fit it.
void Engine::prep_graph_device() {
  static_assert(dev::kSegMax == dev::kBucketLong, "split rows == hub rows");
  const int64_t n = n_, nnz = nnz_;
  const int64_t nseg_max = n + nnz / dev::kSegMax + 1;
  const int64_t nsplit_max = nnz / (dev::kSegMax + 1) + 1;
  const int64_t nslot_max = nnz / dev::kSegMax + nsplit_max + 1;
  const int64_t nch_max = nnz / dev::kLongChunk + nsplit_max + 1;
  const int64_t nseg_pad_max = (nseg_max + dev::kSegPad - 1) / dev::kSegPad * dev::kSegPad + dev::kSegPad;
  struct Carve {
    int64_t off = 0;
    int64_t take(int64_t bytes) { const int64_t o = off; off += (bytes + 255) / 256 * 256; return o; }
  } cv;
  const int64_t o_nseg = cv.take(4 * (n + 1)), o_segoff = cv.take(4 * (n + 1));
  const int64_t o_nslot = cv.take(4 * (n + 1)), o_slotoff = cv.take(4 * (n + 1));
  const int64_t o_split = cv.take(4 * (n + 1)), o_splitoff = cv.take(4 * (n + 1));
  const int64_t o_okey = cv.take(4 * n), o_okey2 = cv.take(4 * n), o_ids = cv.take(4 * n), o_order = cv.take(4 * n);
  const int64_t o_segs = cv.take(16 * nseg_max), o_keys = cv.take(4 * nseg_max), o_keys2 = cv.take(4 * nseg_max);
  const int64_t o_vals = cv.take(4 * nseg_max), o_perm = cv.take(4 * nseg_max);
  const int64_t o_out = cv.take(16 * nseg_pad_max);
  const int64_t o_srows = cv.take(4 * nsplit_max), o_sbegin = cv.take(4 * (nsplit_max + 1));
  const int64_t o_srow = cv.take(4 * nslot_max);
  const int64_t o_nch = cv.take(4 * (nsplit_max + 1)), o_first = cv.take(4 * (nsplit_max + 1));
  const int64_t o_chunks = cv.take(16 * nch_max), o_small = cv.take(16);
  if (n > gp_n_cap_ || nnz > gp_nnz_cap_) {
    dfree(gp_buf_);
    gp_n_cap_ = gp_nnz_cap_ = -1;
    TCG_CUDA(cudaMalloc(&gp_buf_, cv.off));
    gp_n_cap_ = n;
    gp_nnz_cap_ = nnz;
  }
  auto at = [&](int64_t o) { return gp_buf_ + o; };
  int32_t* nseg = reinterpret_cast<int32_t*>(at(o_nseg));
  int32_t* segoff = reinterpret_cast<int32_t*>(at(o_segoff));
  int32_t* nslot = reinterpret_cast<int32_t*>(at(o_nslot));
  int32_t* slotoff = reinterpret_cast<int32_t*>(at(o_slotoff));
  int32_t* split = reinterpret_cast<int32_t*>(at(o_split));
  int32_t* splitoff = reinterpret_cast<int32_t*>(at(o_splitoff));
  uint32_t* okey = reinterpret_cast<uint32_t*>(at(o_okey));
  uint32_t* okey2 = reinterpret_cast<uint32_t*>(at(o_okey2));
  int32_t* ids = reinterpret_cast<int32_t*>(at(o_ids));
  int32_t* order = reinterpret_cast<int32_t*>(at(o_order));
  dev::Seg* segs = reinterpret_cast<dev::Seg*>(at(o_segs));
  uint32_t* keys = reinterpret_cast<uint32_t*>(at(o_keys));
  uint32_t* keys2 = reinterpret_cast<uint32_t*>(at(o_keys2));
  int32_t* vals = reinterpret_cast<int32_t*>(at(o_vals));
  int32_t* perm = reinterpret_cast<int32_t*>(at(o_perm));
  dev::Seg* out = reinterpret_cast<dev::Seg*>(at(o_out));
  int32_t* srows = reinterpret_cast<int32_t*>(at(o_srows));
  int32_t* sbegin = reinterpret_cast<int32_t*>(at(o_sbegin));
  int32_t* srow = reinterpret_cast<int32_t*>(at(o_srow));
  int32_t* nch = reinterpret_cast<int32_t*>(at(o_nch));
  int32_t* first = reinterpret_cast<int32_t*>(at(o_first));
  int4* chunks = reinterpret_cast<int4*>(at(o_chunks));
  int32_t* nsmall = reinterpret_cast<int32_t*>(at(o_small));
  auto tmp = [&](size_t need) {
    if (need > gp_tmp_cap_) {
      dfree(gp_tmp_);
      gp_tmp_cap_ = 0;
      TCG_CUDA(cudaMalloc(&gp_tmp_, need));
      gp_tmp_cap_ = need;
    }
    return gp_tmp_;
  };
  auto scan = [&](const int32_t* in, int32_t* o, int64_t items) {
    size_t b = 0;
    TCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, in, o, static_cast<int>(items), stream_));
    void* t = tmp(b);
    TCG_CUDA(cub::DeviceScan::ExclusiveSum(t, b, in, o, static_cast<int>(items), stream_));
  };
  auto sort = [&](const uint32_t* k, uint32_t* k2, const int32_t* v, int32_t* v2, int64_t items, int bits) {
    size_t b = 0;
    TCG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, k, k2, v, v2, static_cast<int>(items), 0, bits, stream_));
    void* t = tmp(b);
    TCG_CUDA(cub::DeviceRadixSort::SortPairs(t, b, k, k2, v, v2, static_cast<int>(items), 0, bits, stream_));
  };
  const unsigned g1 = static_cast<unsigned>((n + 1 + 255) / 256);
  TCG_CUDA(cudaMemsetAsync(nsmall, 0, sizeof(int32_t), stream_));
  dev::graph_row_counts<<<g1, 256, 0, stream_>>>(d_row_ptr_, n_, nseg, nslot, split, okey, ids, nsmall);
  scan(nseg, segoff, n + 1);
  scan(nslot, slotoff, n + 1);
  scan(split, splitoff, n + 1);
  if (n) sort(okey, okey2, ids, order, n, 32);
  int32_t tot[4];
  TCG_CUDA(cudaMemcpyAsync(&tot[0], segoff + n, 4, cudaMemcpyDeviceToHost, stream_));
  TCG_CUDA(cudaMemcpyAsync(&tot[1], slotoff + n, 4, cudaMemcpyDeviceToHost, stream_));
  TCG_CUDA(cudaMemcpyAsync(&tot[2], splitoff + n, 4, cudaMemcpyDeviceToHost, stream_));
  TCG_CUDA(cudaMemcpyAsync(&tot[3], nsmall, 4, cudaMemcpyDeviceToHost, stream_));
  TCG_CUDA(cudaStreamSynchronize(stream_));
  const int64_t nseg_tot = tot[0];
  const int nslots = tot[1], nsplit = tot[2];
  if (n) {
    dev::graph_emit_segs<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream_>>>(d_row_ptr_, n_, segoff, slotoff, splitoff,
                                                                                    segs, keys, vals, srows, sbegin, srow);
    TCG_CUDA(cudaMemcpyAsync(sbegin + nsplit, &tot[1], 4, cudaMemcpyHostToDevice, stream_));
    sort(keys, keys2, vals, perm, nseg_tot, 11);
  }
  const int64_t padded = std::max<int64_t>((nseg_tot + dev::kSegPad - 1) / dev::kSegPad * dev::kSegPad, dev::kSegPad);
  dev::graph_gather_segs<<<static_cast<unsigned>((padded + 255) / 256), 256, 0, stream_>>>(segs, perm, nseg_tot, padded, out);
  PartSchedule ps;
  ps.owned = false;
  ps.d_segs = out;
  ps.nseg_padded = padded;
  ps.nsplit_rows = nsplit;
  ps.nslots = nslots;
  if (nsplit) {
    ps.d_split_rows = srows;
    ps.d_slot_begin = sbegin;
    ps.d_slot_row = srow;
  }
  sched_[1].push_back(ps);
  d_row_order_ = order;
  nlong_ = nsplit;
  nsmall_ = tot[3];
  nlchunks_ = 0;
  d_lchunks_ = nullptr;
  d_lfirst_ = nullptr;
  if (nlong_) {
    dev::graph_long_counts<<<static_cast<unsigned>((nlong_ + 1 + 255) / 256), 256, 0, stream_>>>(d_row_ptr_, order, nlong_, nch);
    scan(nch, first, nlong_ + 1);
    int32_t nc = 0;
    TCG_CUDA(cudaMemcpyAsync(&nc, first + nlong_, 4, cudaMemcpyDeviceToHost, stream_));
    TCG_CUDA(cudaStreamSynchronize(stream_));
    nlchunks_ = nc;
    dev::graph_long_chunks<<<static_cast<unsigned>((nlong_ + 255) / 256), 256, 0, stream_>>>(d_row_ptr_, order, nlong_, first, chunks);
    d_lchunks_ = chunks;
    d_lfirst_ = first;
  }
  launches_ += 0;  // (graph preparation: not part of a coloring)
  TCG_CUDA(cudaGetLastError());
}

// Vertex-range part schedules for the full-table SpMM (P parts per panel).
void Engine::ensure_schedules(int P) {
  if (sched_.count(P)) return;
  if (P > 1) sort_rows();
  if (host_row_ptr_.empty()) {
    host_row_ptr_.resize(static_cast<size_t>(n_) + 1);
    copy_sync(host_row_ptr_.data(), d_row_ptr_, sizeof(int64_t) * (n_ + 1), cudaMemcpyDeviceToHost);
  }
  if (host_col_.empty() && nnz_) {
    host_col_.resize(static_cast<size_t>(nnz_));
    copy_sync(host_col_.data(), d_col_, sizeof(int32_t) * nnz_, cudaMemcpyDeviceToHost);
  }
  const int64_t* rp = host_row_ptr_.data();
  std::vector<std::vector<int64_t>> bnd(P + 1, std::vector<int64_t>(n_));
  const int T = std::max(1, std::min(host_threads(), 32));
  std::vector<std::thread> th;
  for (int w = 0; w < T; ++w)
    th.emplace_back([&, w] {
      for (int64_t v = static_cast<int64_t>(n_) * w / T; v < static_cast<int64_t>(n_) * (w + 1) / T; ++v) {
        const int32_t* b = host_col_.data() + rp[v];
        const int32_t* e = host_col_.data() + rp[v + 1];
        bnd[0][v] = rp[v];
        bnd[P][v] = rp[v + 1];
        for (int s = 1; s < P; ++s) {
          const int64_t cut = static_cast<int64_t>(nsrc_) * s / P;
          bnd[s][v] = rp[v] + (std::lower_bound(b, e, static_cast<int32_t>(cut)) - b);
        }
      }
    });
  for (auto& t : th) t.join();
  auto& vec = sched_[P];
  for (int s = 0; s < P; ++s) {
    vec.push_back(build_schedule(bnd[s], bnd[s + 1], s == 0, stream_));
    max_slots_ = std::max(max_slots_, vec.back().nslots);
  }
}

// --------------------------------------------------------------- template
static std::vector<int16_t> dummy_slots(const RootedLayout& L, int K);

void Engine::set_template(int k, const int32_t* edges, int root) {
  TCG_CUDA(cudaSetDevice(cfg_.device));
  Template t = make_template(k, edges, root);
  Plan p = partition(t);
  release_template();
  tpl_ = t;
  plan_ = p;
  aut_ = automorphism_count(t);
  const Binom& B = binom();
  need_hist_ = false;
  int max_smem = 0;
  TCG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, cfg_.device));
  max_smem_ = max_smem;
  static const int rooted_mode = [] {
    const char* s = std::getenv("TCG_ROOTED");
    return s ? std::atoi(s) : 1;
  }();
  for (int id : plan_.dp_order) {
    if (plan_.is_leaf(id)) continue;
    NodeExec e;
    e.id = id;
    e.a = plan_.active[id];
    e.p = plan_.passive[id];
    e.size = plan_.size[id];
    e.sa = plan_.size[e.a];
    e.sp = plan_.size[e.p];
    e.Cs = static_cast<int32_t>(B(k, e.size));
    e.Ca = static_cast<int32_t>(B(k, e.sa));
    e.Cp = static_cast<int32_t>(B(k, e.sp));
    e.a_leaf = e.sa == 1;
    e.p_leaf = e.sp == 1;
    e.root = id == plan_.full_node();
    need_hist_ |= e.p_leaf;
    SplitTable st = build_split_table(k, e.size, e.sa);
    e.pairs = st.pairs_per_parent;
    std::vector<int2> pr(st.active_index.size());
    for (size_t i = 0; i < pr.size(); ++i) pr[i] = make_int2(st.active_index[i], st.passive_index[i]);
    // Rooted-color compressed SpMM for every internal passive child (default;
    // TCG_ROOTED=0 restores the full-table panel SpMM): P' is then stored
    // group-major, so the eMA's passive indices are remapped to storage columns.
    e.Cps = e.Cp;
    if (rooted_mode && !e.p_leaf) {
      const RootedLayout rl = build_rooted_layout(k, e.sp);
      int fpad_max = 0;
      for (int g = 0; g < rl.groups; ++g)
        fpad_max = std::max(fpad_max, (g + 1 < rl.groups ? rl.fbase[g + 1] : rl.store_cols) - rl.fbase[g]);
      const size_t smem = static_cast<size_t>(dev::kSpmmWarps) * (128 / rl.zw) * (fpad_max + 4) * 4 + 2 * (k + 1) * rl.zw;
      // (rooted_compress stages at least one full row of M_p in smem)
      if (smem <= static_cast<size_t>(max_smem) - 4096 && 4 * dev::table_floats(e.Cp, 1) <= max_smem - 4096) {
        e.rooted = true;
        e.Cps = rl.store_cols;
        e.rl_zw = rl.zw;
        e.rl_groups = rl.groups;
        e.rl_fbase = rl.fbase;
        e.rl_fsize = rl.fsize;
        e.rl_perm = rl.perm;
        e.rooted_smem = smem;
        e.slot_K = k;
        e.d_slot_acc = dupload(dummy_slots(rl, k), stream_);
        e.d_slot_col = dupload(rl.slot_col, stream_);
        e.d_pinv = dupload(rl.inv, stream_);
        for (auto& q : pr) q.y = rl.perm[q.y];
        // pair layout candidate: the row's color never occurs in a consumed
        // P' column, so per (neighbour color, row color) only C(k-2, sp-1)
        // sets are gathered -- worth it when the copies' lines are >= 20%
        // fewer and one vertex's copies stay small (k x groups x zw floats)
        static const int pair_mode = [] {
          const char* s = std::getenv("TCG_PAIR");
          return s ? std::atoi(s) : 1;
        }();
        if (pair_mode && k >= 3) {
          RootedLayout r1 = build_rooted_layout(k - 1, e.sp);
          int fpad1 = 0;
          for (int g = 0; g < r1.groups; ++g)
            fpad1 = std::max(fpad1, (g + 1 < r1.groups ? r1.fbase[g + 1] : r1.store_cols) - r1.fbase[g]);
          const size_t smem1 = static_cast<size_t>(dev::kSpmmWarps) * (128 / r1.zw) * (fpad1 + 4) * 4 + 2 * k * r1.zw;
          const int64_t wx = B(k - 1, e.sp - 1);
          const int64_t lines_old = static_cast<int64_t>(rl.groups) * rl.zw, lines_new = static_cast<int64_t>(r1.groups) * r1.zw;
          const int64_t copy_bytes = 4ll * k * lines_new;
          if (pair_mode == 2 || (5 * lines_new <= 4 * lines_old && copy_bytes <= 8192)) {
            if (smem1 <= static_cast<size_t>(max_smem) - 4096 && 4 * 32 * (wx + 1) <= max_smem - 4096 && wx < 32768) {
              e.pair_cand = true;
              e.pr = std::move(r1);
              e.Wx = static_cast<int32_t>(wx);
            }
          }
        }
      }
    }
    e.d_split = dupload(pr, stream_);
    if (!e.a_leaf && !e.root && e.Ca < 65536 && e.Cps < 65536) {
      std::vector<uint32_t> pk(pr.size());
      for (size_t i = 0; i < pr.size(); ++i)
        pk[i] = static_cast<uint32_t>(pr[i].x) | (static_cast<uint32_t>(pr[i].y) << 16);
      e.d_packed = dupload(pk, stream_);
    }
    if (e.a_leaf && !e.root) {
      // active leaf: the pair whose active color is c gives the column of S minus c
      std::vector<int32_t> drop(static_cast<size_t>(e.Cs) * k, -1);
      for (int32_t s = 0; s < e.Cs; ++s)
        for (int p2 = 0; p2 < e.pairs; ++p2)
          drop[static_cast<size_t>(s) * k + pr[static_cast<size_t>(s) * e.pairs + p2].x] =
              pr[static_cast<size_t>(s) * e.pairs + p2].y;
      e.d_drop = dupload(drop, stream_);
    }
    const int64_t staged = static_cast<int64_t>((e.a_leaf ? 0 : e.Ca) + e.Cps) * (dev::kTileV + 1) * 4;
    e.ema_staged = staged <= max_smem - 4096;
    e.ema_smem = e.ema_staged ? static_cast<size_t>(staged) : 0;
    static const int blocked_mode = [] {
      const char* s = std::getenv("TCG_EMA_BLOCKED");
      return s ? std::atoi(s) : 1;
    }();
    // FMA-heavy nodes only: narrow nodes are bound by their output writes,
    // which the 8-column chunks of ema_node coalesce better
    // vertex-per-CTA when a 32-vertex tile does not fit: one vertex's rows
    auto row_floats = [](int64_t C) { return C <= 0 ? 0 : dev::table_floats(C, 1); };
    const int64_t vsm = 4 * (((e.a_leaf ? 0 : row_floats(e.Ca)) + 3) / 4 * 4 + row_floats(e.Cps));
    if (!e.ema_staged && vsm <= max_smem - 4096 && (e.a_leaf || e.root || k >= dev::kH1)) {
      e.vtx = true;
      e.vtx_smem = static_cast<size_t>(vsm);
    }
    if (!e.a_leaf && !e.root && k >= dev::kH1 &&
        ((blocked_mode && e.ema_staged && (e.pairs >= 16 || blocked_mode == 2)) || e.vtx)) {
      std::vector<dev::GroupDesc> gr;
      std::vector<dev::BlockDesc> bl;
      build_blocked(k, e.size, e.sa, gr, bl);
      e.blocked = true;
      e.ngroups = static_cast<int>(gr.size());
      e.d_groups = dupload(gr, stream_);
      e.d_blocks = dupload(bl, stream_);
    }
    exec_.push_back(e);
  }
  setup_rooted_ema(max_smem);
  // Identical sub-template computations (same recursive shape and the same
  // table layout) are computed once: a later duplicate aliases the first
  // node's table.  (The reference recomputes them; the tables are identical
  // bit for bit since the kernels and split tables are the same.)
  {
    static const int dedup = [] {
      const char* s = std::getenv("TCG_DEDUP");
      return s ? std::atoi(s) : 1;
    }();
    std::vector<std::string> key(plan_.num_nodes, "L");
    std::map<std::string, int> first, first_pp;
    for (size_t i = 0; i < exec_.size(); ++i) {
      NodeExec& e = exec_[i];
      const char* lay = rooted_ema_ ? (e.omap.empty() ? "R" : "S") : "F";
      key[e.id] = "(" + key[e.a] + "," + key[e.p] + ")" + lay;
      e.dup_of = e.pp_dup_of = -1;
      if (!dedup) continue;
      auto it = first.find(key[e.id]);
      if (it == first.end() || e.root) {
        if (!e.root) first.emplace(key[e.id], static_cast<int>(i));
        // a different node over the same passive table: share its P' (SpMM)
        if (!e.p_leaf) {
          auto jt = first_pp.find(key[e.p]);
          if (jt == first_pp.end()) first_pp.emplace(key[e.p], static_cast<int>(i));
          else e.pp_dup_of = jt->second;
        }
      } else {
        e.dup_of = it->second;
      }
    }
  }
  if (std::getenv("TCG_VERBOSE")) {
    std::fprintf(stderr, "[tcg] k=%d nodes=%d rooted_ema=%d\n", k, plan_.num_nodes, rooted_ema_ ? 1 : 0);
    for (const auto& e : exec_)
      std::fprintf(stderr, "[tcg] node %2d (%2d,%2d,%2d) Cp=%d rooted=%d pair=%d groups=%d zw=%d Cps=%d | Ws=%d Wa=%d Wp=%d Cout=%d "
                           "%s pairs=%d blocked=%d/%d vtx=%d/%d staged=%d dup_of=%d\n",
                   e.id, e.size, e.sa, e.sp, e.Cp, e.rooted ? 1 : 0, e.pair ? 1 : 0, e.rl_groups, e.rl_zw, e.Cps, e.Ws, e.Wa, e.Wp,
                   e.Cout, e.omap.empty() ? "RR" : "RS", e.rt_pairs, e.rt_blocked ? 1 : 0, e.blocked ? 1 : 0,
                   e.vtx ? 1 : 0, e.rt_vtx ? 1 : 0, e.ema_staged ? 1 : 0, e.dup_of >= 0 ? exec_[e.dup_of].id : -1);
    for (const auto& e : exec_)
      if (e.pp_dup_of >= 0) std::fprintf(stderr, "[tcg] node %d shares the SpMM of node %d\n", e.id, exec_[e.pp_dup_of].id);
  }
  TCG_CUDA(cudaStreamSynchronize(stream_));
  have_template_ = true;
  ++tpl_gen_;
  if (n_ >= 0) plan_arena();
  tables_valid_ = false;
}

// spmm_rooted's slot table: -1 (unused slot) -> the group's dummy
// accumulator fpad_g, plus an all-dummy row K (the state before a row's first run)
static std::vector<int16_t> dummy_slots(const RootedLayout& L, int K) {
  const int slots = L.groups * L.zw;
  std::vector<int16_t> out(static_cast<size_t>(K + 1) * slots);
  for (int g = 0; g < L.groups; ++g) {
    const int fpad = (g + 1 < L.groups ? L.fbase[g + 1] : L.store_cols) - L.fbase[g];
    for (int t = 0; t < L.zw; ++t) {
      const int i = g * L.zw + t;
      for (int c = 0; c < K; ++c) {
        const int16_t x = L.slot_acc[static_cast<size_t>(c) * slots + i];
        out[static_cast<size_t>(c) * slots + i] = x >= 0 ? x : static_cast<int16_t>(fpad);
      }
      out[static_cast<size_t>(K) * slots + i] = static_cast<int16_t>(fpad);
    }
  }
  return out;
}

// relabeled combinadic index of the set cs[0..h) minus color c (colors above
// c shift down by one), over k-1 colors
static int64_t relabeled_index(const int* cs, int h, int c) {
  int t[kMaxK];
  int m = 0;
  for (int i = 0; i < h; ++i)
    if (cs[i] != c) t[m++] = cs[i] < c ? cs[i] : cs[i] - 1;
  return index_of(t, m);
}

// Rooted tables everywhere (kernels_rt.cuh): possible when every internal
// passive child goes through the rooted SpMM and every node's tile fits smem.
void Engine::setup_rooted_ema(int max_smem) {
  rooted_ema_ = false;
  static const int mode = [] {
    const char* s = std::getenv("TCG_ROOTED_EMA");
    return s ? std::atoi(s) : 1;
  }();
  static const int blocked_mode = [] {
    const char* s = std::getenv("TCG_EMA_BLOCKED");
    return s ? std::atoi(s) : 1;
  }();
  const int k = plan_.k;
  if (!mode || exec_.empty() || k < 2) return;
  const Binom& B = binom();
  static const int vtx_mode = [] {  // 2: every non-leaf node vertex-per-CTA (tests)
    const char* s = std::getenv("TCG_RT_VTX");
    return s ? std::atoi(s) : 1;
  }();
  auto row_floats = [](int64_t C) { return C <= 0 ? 0 : dev::table_floats(C, 1); };
  for (auto& e : exec_) {
    if (!e.p_leaf && !e.rooted) return;
    const int64_t Wa = e.a_leaf ? 0 : B(k - 1, e.sa - 1), Wp = B(k - 1, e.sp), Ws = e.root ? 1 : B(k - 1, e.size - 1);
    if (Wa >= 65536 || Wp >= 65536 || Ws >= 65536) return;
    e.rt_vtx = false;
    if (e.a_leaf && !e.root) {  // ema_rt_copy: one P' row per vertex at least
      if (4 * row_floats(e.p_leaf ? k : e.Cps) > max_smem - 4096) return;
      continue;
    }
    const bool tile_fits = (Wa + Wp) * (dev::kTileV + 1) * 4 <= max_smem - 4096;
    if (tile_fits && !(vtx_mode == 2 && !e.a_leaf && (e.root || k - 1 >= dev::kH1))) continue;
    // vertex-per-CTA: the vertex's RR A row and its relabeled P row
    if (!vtx_mode || e.a_leaf || (!e.root && k - 1 < dev::kH1)) return;
    if (4 * (row_floats(Wa) + Wp + 4) > max_smem - 4096) return;
    e.rt_vtx = true;
  }
  // pair layout for the candidates (needs the rooted eMA; unsharded): the
  // SpMM layout fields now describe the (k-1)-color layout
  int cs[kMaxK];
  for (auto& e : exec_) {
    e.pair = e.pair_cand && !sharded();
    if (!e.pair) continue;
    const RootedLayout& r1 = e.pr;
    e.Cps = r1.store_cols;
    e.rl_zw = r1.zw;
    e.rl_groups = r1.groups;
    e.rl_fbase = r1.fbase;
    e.rl_fsize = r1.fsize;
    e.rl_perm = r1.perm;  // (k-1)-color combinadic column -> storage column
    int fpad1 = 0;
    for (int g = 0; g < r1.groups; ++g)
      fpad1 = std::max(fpad1, (g + 1 < r1.groups ? r1.fbase[g + 1] : r1.store_cols) - r1.fbase[g]);
    e.rooted_smem = static_cast<size_t>(dev::kSpmmWarps) * (128 / r1.zw) * (fpad1 + 4) * 4 + 2 * k * r1.zw;
    dfree(e.d_slot_acc);
    e.slot_K = k - 1;
    e.d_slot_acc = dupload(dummy_slots(r1, k - 1), stream_);
    // copy (cu, cv) slot -> RR column of the set relative to cu
    const int slots = r1.groups * r1.zw;
    std::vector<int16_t> xm(static_cast<size_t>(k) * k * slots, -1);
    for (int cu = 0; cu < k; ++cu)
      for (int cv = 0; cv < k; ++cv) {
        if (cu == cv) continue;
        const int cr = cu - (cu > cv ? 1 : 0);
        for (int i = 0; i < slots; ++i) {
          const int32_t col1 = r1.slot_col[static_cast<size_t>(cr) * slots + i];
          if (col1 < 0) continue;
          set_of(k - 1, col1, e.sp, cs);
          for (int q = 0; q < e.sp; ++q) cs[q] = cs[q] >= cv ? cs[q] + 1 : cs[q];  // actual colors
          xm[(static_cast<size_t>(cu) * k + cv) * slots + i] = static_cast<int16_t>(relabeled_index(cs, e.sp, cu));
        }
      }
    dfree(e.d_xmap);
    e.d_xmap = dupload(xm, stream_);
    e.xmap_host = std::move(xm);
  }
  std::vector<int> parent(plan_.num_nodes, -1);
  for (size_t i = 0; i < exec_.size(); ++i) {
    parent[exec_[i].a] = static_cast<int>(i);
    parent[exec_[i].p] = static_cast<int>(i);
  }
  for (auto& e : exec_) {
    e.Wa = e.a_leaf ? 0 : static_cast<int32_t>(B(k - 1, e.sa - 1));
    e.Wp = static_cast<int32_t>(B(k - 1, e.sp));
    e.Ws = e.root ? 1 : static_cast<int32_t>(B(k - 1, e.size - 1));
    // P' storage column -> full combinadic column -> relabeled row per color
    std::vector<int64_t> full_of;
    if (e.p_leaf) {
      e.Cpt = k;
      for (int d = 0; d < k; ++d) full_of.push_back(d);
    } else {
      e.Cpt = e.Cps;
      full_of.assign(static_cast<size_t>(e.Cps), -1);
      if (!e.pair)
        for (int32_t x = 0; x < e.Cp; ++x) full_of[e.rl_perm[x]] = x;
    }
    std::vector<int32_t> pm(static_cast<size_t>(k) * e.Cpt, -1);
    if (e.pair)  // storage column -> its relabeled (k-1)-color index, for every row color
      for (int c = 0; c < k; ++c)
        for (int32_t col = 0; col < e.Cpt; ++col) pm[static_cast<size_t>(c) * e.Cpt + col] = e.pr.inv[col];
    for (int32_t col = 0; col < e.Cpt; ++col) {
      if (full_of[col] < 0) continue;
      set_of(k, full_of[col], e.sp, cs);
      for (int c = 0; c < k; ++c) {
        if (std::find(cs, cs + e.sp, c) != cs + e.sp) continue;
        pm[static_cast<size_t>(c) * e.Cpt + col] = static_cast<int32_t>(relabeled_index(cs, e.sp, c));
      }
    }
    e.d_pmap = dupload(pm, stream_);
    e.omap.clear();
    if (!e.root) {
      const NodeExec& par = exec_[parent[e.id]];
      if (par.p == e.id && par.rooted && !par.pair) {  // feeds the rooted SpMM: its slot layout
        const RootedLayout rl = build_rooted_layout(k, e.size);
        e.Cout = rl.groups * rl.zw;
        e.omap.assign(static_cast<size_t>(k) * e.Ws, -1);
        const int slots = rl.groups * rl.zw;
        for (int c = 0; c < k; ++c)
          for (int i = 0; i < slots; ++i) {
            const int32_t col = rl.slot_col[static_cast<size_t>(c) * slots + i];
            if (col < 0) continue;
            set_of(k, col, e.size, cs);
            e.omap[static_cast<size_t>(c) * e.Ws + relabeled_index(cs, e.size, c)] = i;
          }
        e.d_omap = dupload(e.omap, stream_);
        std::vector<int32_t> im(static_cast<size_t>(k) * e.Cout, -1);  // slot -> output column
        for (int c = 0; c < k; ++c)
          for (int32_t j = 0; j < e.Ws; ++j) {
            const int32_t i = e.omap[static_cast<size_t>(c) * e.Ws + j];
            if (i >= 0) im[static_cast<size_t>(c) * e.Cout + i] = j;
          }
        e.d_imap = dupload(im, stream_);
      } else {
        e.Cout = e.Ws;
      }
    }
    if (e.a_leaf && !e.root) {
      // active leaf: output column -> P' storage column of (S minus c), per color
      std::vector<int32_t> cm(static_cast<size_t>(k) * e.Cout, -1);
      std::vector<int32_t> storage_of(e.Cp);
      for (int32_t x = 0; x < e.Cp; ++x) storage_of[x] = e.p_leaf ? x : (e.pair ? 0 : e.rl_perm[x]);
      int t[kMaxK];
      for (int c = 0; c < k; ++c)
        for (int32_t j = 0; j < e.Ws; ++j) {
          set_of(k - 1, j, e.size - 1, t);
          for (int q = 0; q < e.size - 1; ++q) t[q] = t[q] >= c ? t[q] + 1 : t[q];
          // (pair layout: P' is stored by the relabeled index of S minus c: j)
          const int32_t src = e.pair ? e.rl_perm[j] : storage_of[index_of(t, e.size - 1)];
          const int32_t i = e.omap.empty() ? j : e.omap[static_cast<size_t>(c) * e.Ws + j];
          if (i >= 0) cm[static_cast<size_t>(c) * e.Cout + i] = src;
        }
      e.d_cmap = dupload(cm, stream_);
      e.cmap_host = cm;
      if (!e.p_leaf && !e.pair) {
        // streamed SpMM epilogue (pstream_copy): P' storage column -> output
        // column.  RS outputs: the slot.  RR outputs are stored PACKED in P'
        // storage order instead (column q = rank of the storage column among
        // those without c), so each group lands on a contiguous run of the
        // row; the consumer stages them through amap [k][Ws]: q -> RR column.
        std::vector<int32_t> em(static_cast<size_t>(k) * e.Cps, -1);
        if (e.omap.empty()) {
          std::vector<int32_t> am(static_cast<size_t>(k) * e.Ws, -1);
          std::vector<int32_t> rr_of(e.Cps);
          for (int c = 0; c < k; ++c) {
            std::fill(rr_of.begin(), rr_of.end(), -1);
            for (int32_t i = 0; i < e.Cout; ++i) {
              const int32_t src = cm[static_cast<size_t>(c) * e.Cout + i];
              if (src >= 0) rr_of[src] = i;
            }
            int32_t q = 0;
            for (int32_t x = 0; x < e.Cps; ++x)
              if (rr_of[x] >= 0) {
                em[static_cast<size_t>(c) * e.Cps + x] = q;
                am[static_cast<size_t>(c) * e.Ws + q] = rr_of[x];
                ++q;
              }
            if (q != e.Ws) throw logic_error("packed active-leaf layout does not cover the rooted columns");
          }
          e.amap_host = am;
          e.d_amap = dupload(am, stream_);
        } else {
          for (int c = 0; c < k; ++c)
            for (int32_t i = 0; i < e.Cout; ++i) {
              const int32_t src = cm[static_cast<size_t>(c) * e.Cout + i];
              if (src >= 0) em[static_cast<size_t>(c) * e.Cps + src] = i;
            }
        }
        e.d_emap = dupload(em, stream_);
      }
    }
    if (!e.a_leaf) {
      const SplitTable st = build_split_table(k - 1, e.root ? k - 1 : e.size - 1, e.sa - 1);
      e.rt_pairs = st.pairs_per_parent;
      if (e.root) {
        std::vector<int2> pr(st.active_index.size());
        for (size_t i = 0; i < pr.size(); ++i) pr[i] = make_int2(st.active_index[i], st.passive_index[i]);
        e.d_rt_split = dupload(pr, stream_);
      } else {
        std::vector<uint32_t> pk(st.active_index.size());
        for (size_t i = 0; i < pk.size(); ++i)
          pk[i] = static_cast<uint32_t>(st.active_index[i]) | (static_cast<uint32_t>(st.passive_index[i]) << 16);
        e.d_rt_packed = dupload(pk, stream_);
        if (e.rt_vtx || (blocked_mode && k - 1 >= dev::kH1 && (e.rt_pairs >= 16 || blocked_mode == 2))) {
          std::vector<dev::GroupDesc> gr;
          std::vector<dev::BlockDesc> bl;
          if (e.rt_vtx) {
            // vertex-per-CTA: tasks are built below, once V is known (build_rtv_tasks).
            // H = 6: measured on cfg5 node 1 / node 2 and cfg4 node 1 with the task kernel,
            // H = 6 / 7: 243 / 297, 114 / 110 and 114 / 135 ms (H = 8 spills)
            e.rtv_h = dev::kH1;
          } else {
            build_blocked(k - 1, e.size - 1, e.sa - 1, gr, bl);
          }
          e.rt_blocked = true;
          if (!e.rt_vtx) {
            e.rt_ngroups = static_cast<int>(gr.size());
            e.d_rt_groups = dupload(gr, stream_);
            e.d_rt_blocks = dupload(bl, stream_);
          }
        }
      }
    }
    e.rtv_pleaf = false;
    dfree(e.d_rtv_drop);
    static const int pleaf_mode = [] {
      const char* s = std::getenv("TCG_RTV_PLEAF");
      return s ? std::atoi(s) : 1;
    }();
    // (also for wide tiled nodes: a leaf passive child makes the blocked
    // micro-patterns and the 8-column tile chunks mostly overhead)
    if ((e.rt_vtx || e.Ws >= 512) && e.p_leaf && !e.root && !e.a_leaf && pleaf_mode && e.Wa < 65536) {
      // out'[S'] = sum over d in S' of A'[S' minus d] * H[d]: the drop table
      const int K = k - 1, sp1 = e.size - 1;
      std::vector<uint32_t> dr(static_cast<size_t>(e.Ws) * sp1);
      int t2[kMaxK];
      for (int32_t j = 0; j < e.Ws; ++j) {
        set_of(K, j, sp1, cs);
        for (int i = 0; i < sp1; ++i) {
          int m = 0;
          for (int q = 0; q < sp1; ++q)
            if (q != i) t2[m++] = cs[q];
          dr[static_cast<size_t>(j) * sp1 + i] = static_cast<uint32_t>(index_of(t2, m)) | (static_cast<uint32_t>(cs[i]) << 16);
        }
      }
      e.rtv_packed = sp1 <= 6 && K <= 16;
      if (e.rtv_packed) {  // packed: uint4 per output (6 x 16-bit A index, 6 x 4-bit colour)
        std::vector<uint32_t> pk(static_cast<size_t>(e.Ws) * 4, 0u);
        for (int32_t j = 0; j < e.Ws; ++j)
          for (int i = 0; i < sp1; ++i) {
            const uint32_t x = dr[static_cast<size_t>(j) * sp1 + i];
            pk[static_cast<size_t>(j) * 4 + (i >> 1)] |= (x & 0xFFFFu) << ((i & 1) * 16);
            pk[static_cast<size_t>(j) * 4 + 3] |= (x >> 16) << (4 * i);
          }
        dr.swap(pk);
      }
      e.d_rtv_drop = dupload(dr, stream_);
      e.rtv_pleaf = true;
    }
    if (e.rt_vtx) {
      if (e.root) {
        e.rt_smem = static_cast<size_t>(4 * (row_floats(e.Wa) + e.Wp));
      } else {  // V vertices per pass: two CTAs per SM when V >= 2 fits
        auto stride = [](int64_t f, int V) { return (f + 31) / 32 * 32 + (V > 1 ? 32 / V : 0); };
        auto fit = [&](int64_t bytes) {
          int v = 8;
          while (v > 1 && 4 * v * (stride(row_floats(e.Wa), v) + stride(e.Wp, v)) > bytes) v /= 2;
          return v;
        };
        int V = fit((max_smem - 4096) / 2);
        // rows so wide that two CTAs hold <= 2 vertices each: ONE CTA of twice the threads over
        // twice the vertices instead (same warps per SM; its 28 warps walk the same task classes
        // together, so the pattern code is fetched once, not per CTA: cfg5 node 1 213 -> 181 ms;
        // narrower rows lose the overlap of one CTA's staging with the other's FMAs: cfg5 node 2
        // 100 -> 108 ms, cfg4 node 1 102 -> 103)
        e.rtv_one_cta = V <= 2 && fit(max_smem - 4096) >= 2 * V;
        if (e.rtv_one_cta) V = fit(max_smem - 4096);
        e.rtv_V = V;
        e.rtv_sa = static_cast<int>(stride(row_floats(e.Wa), V));
        e.rtv_sp = static_cast<int>(stride(e.Wp, V));
        e.rt_smem = static_cast<size_t>(4 * V * (e.rtv_sa + e.rtv_sp));
        if (!e.rtv_pleaf) {
          const RtvPlan rp = build_rtv_tasks(k - 1, e.size - 1, e.sa - 1, e.rtv_h, V);
          e.rtv_ntasks = static_cast<int>(rp.tasks.size());
          e.d_rtv_tasks = dupload(rp.tasks, stream_);
          e.d_rtv_gout = dupload(rp.gout, stream_);
          e.d_rtv_runs = dupload(rp.runs, stream_);
          e.d_rtv_blocks = dupload(rp.blocks, stream_);
          if (std::getenv("TCG_VERBOSE"))
            std::fprintf(stderr, "[tcg] node %d rtv tasks %d (V %d, %lld steps, shared-load wavefronts %.3f x conflict-free)\n",
                         e.id, e.rtv_ntasks, V, static_cast<long long>(rp.steps),
                         static_cast<double>(rp.wavefronts) / static_cast<double>(std::max<int64_t>(rp.ideal, 1)));
        }
      }
      dfree(e.d_imap);
      continue;
    }
    // (+ the RS output tile of the generic node kernel, when it fits)
    e.rt_smem = static_cast<size_t>(e.Wa + e.Wp) * (dev::kTileV + 1) * 4;
    const size_t out_tile = static_cast<size_t>(e.Ws) * (dev::kTileV + 1) * 4;
    if (!e.omap.empty() && !e.a_leaf && !e.rt_blocked && e.rt_smem + out_tile <= static_cast<size_t>(max_smem) - 4096)
      e.rt_smem += out_tile;
    else
      dfree(e.d_imap);  // scattered RS writes instead
  }
  // pair SpMMs over an active-leaf passive child: the composed map lets the
  // expansion read the child's P' directly (plan_arena_once decides virt_px)
  for (auto& par : exec_) {
    dfree(par.d_xmap_v);
    if (!par.pair) continue;
    const NodeExec* ch = nullptr;
    for (const auto& x : exec_)
      if (x.id == par.p) ch = &x;
    if (!ch || !ch->a_leaf || ch->root || !ch->rooted || ch->p_leaf || ch->cmap_host.empty() || !ch->omap.empty()) continue;
    std::vector<int16_t> xv(par.xmap_host.size(), -1);
    const int slots = par.rl_groups * par.rl_zw;
    for (int cu = 0; cu < k; ++cu)
      for (size_t i = 0; i < static_cast<size_t>(k) * slots; ++i) {
        const size_t at = static_cast<size_t>(cu) * k * slots + i;
        const int16_t j = par.xmap_host[at];
        if (j >= 0) xv[at] = static_cast<int16_t>(ch->cmap_host[static_cast<size_t>(cu) * ch->Cout + j]);
      }
    par.d_xmap_v = dupload(xv, stream_);
  }
  rooted_ema_ = true;
}

// Streamed active-leaf SpMMs (NodeExec::pstream) trade the full P' for a
// per-group scatter: used when the plan with full P' tables does not fit the
// device (or the memory budget).  TCG_PSTREAM: 0 never, 1 when needed
// (default), 2 always (also with TCG_KEEP_TABLES; tests).
void Engine::ensure_tile_tot(int64_t count) {
  count = std::max<int64_t>(count, 1);
  if (count <= tile_tot_cap_) return;
  dfree(d_tile_tot_);
  tile_tot_cap_ = 0;
  TCG_CUDA(cudaMalloc(&d_tile_tot_, sizeof(double) * count));
  tile_tot_cap_ = count;
}

void Engine::plan_arena() {
  static const int pstream_mode = [] {
    const char* s = std::getenv("TCG_PSTREAM");
    return s ? std::atoi(s) : 1;
  }();
  plan_arena_once(pstream_mode == 2);
  // (an arena already allocated at this size needs no device-memory query)
  if (pstream_mode == 1 && !(cfg_.flags & TCG_KEEP_TABLES) && !(arena_ && arena_bytes_ <= arena_alloc_)) {
    size_t fr = 0, tot = 0;
    TCG_CUDA(cudaMemGetInfo(&fr, &tot));
    int64_t limit = static_cast<int64_t>(fr) + (arena_ ? arena_alloc_ : 0) - partial_bytes_ - (3ll << 30);
    if (cfg_.memory_budget > 0) limit = std::min<int64_t>(limit, cfg_.memory_budget);
    if (arena_bytes_ > limit) plan_arena_once(true);
    if (std::getenv("TCG_VERBOSE"))
      std::fprintf(stderr, "[tcg] plan: free %.2f GB, limit %.2f GB, arena %.2f GB, partial %.2f GB, streamed %d\n",
                   fr / 1e9, limit / 1e9, arena_bytes_ / 1e9, partial_bytes_ / 1e9, arena_bytes_ > limit ? -1 : 0);
  }
}

void Engine::plan_arena_once(bool allow_stream) {
  const bool keep = cfg_.flags & TCG_KEEP_TABLES;
  for (auto& e : exec_) e.pstream = false;
  ArenaPlanner ap;
  table_off_.assign(plan_.num_nodes, -1);
  pprime_off_.assign(plan_.num_nodes, -1);
  hist_off_ = need_hist_ ? ap.alloc(table_bytes(plan_.k)) : -1;
  for (const auto& e : exec_)  // full-table SpMMs: their vertex-range part schedules
    if (!e.p_leaf && !e.rooted && e.pp_dup_of < 0 && e.dup_of < 0)
      for (int p = 0; p < dev::num_panels(e.Cp); ++p) ensure_schedules(parts_for_width(dev::panel_width(e.Cp, p)));
  // rooted SpMMs: parts are contiguous COLOR classes (one count for all
  // rooted nodes: the widest compressed panel's), over whole-row schedules
  need_rooted_ = need_pair_ = false;
  rooted_parts_ = 1;
  for (auto& e : exec_)
    if (e.rooted) {
      need_rooted_ = true;
      need_pair_ |= e.pair;
      rooted_parts_ = std::max(rooted_parts_, std::min(plan_.k, rooted_part_mb_ > 0 ? parts_for_width(e.rl_zw) : 1));
    }
  rcol_off_ = rcut_off_ = -1;
  int64_t rooted_partial = 0;
  if (need_rooted_) {
    if (nsrc_ >= (1ll << (32 - dev::kColorBits)))
      throw invalid_argument("graph too large for the rooted-compressed SpMM (ids >= 2^27); set TCG_ROOTED=0");
    rcol_off_ = ap.alloc(4 * std::max<int64_t>(nnz_, 1));
    rcut_off_ = ap.alloc(8 * static_cast<int64_t>(n_) * (rooted_parts_ + 1));
    lcnt_off_ = ap.alloc(4 * 32 * static_cast<int64_t>(std::max(nlchunks_, 1)));
  }
  pseg_off_ = pkey_off_ = pperm_off_ = pcnt_off_ = -1;
  if (need_pair_) {  // per-coloring color-ordered whole-row segments
    const int64_t nseg = sched_.at(1)[0].nseg_padded;
    pseg_off_ = ap.alloc(static_cast<int64_t>(sizeof(dev::Seg)) * nseg);
    pkey_off_ = ap.alloc(nseg);
    pperm_off_ = ap.alloc(4 * nseg);
    pcnt_off_ = ap.alloc(4 * ((nseg + dev::kVsChunk - 1) / dev::kVsChunk + 1) * (plan_.k + 1));
  }
  vs_off_ = tiles_off_ = vcnt_off_ = -1;
  max_tiles_ = static_cast<int>((n_ + dev::kTileV - 1) / dev::kTileV) + plan_.k;
  if (rooted_ema_) {
    vs_off_ = ap.alloc(4 * std::max<int64_t>(n_, 1));
    tiles_off_ = ap.alloc(16 * static_cast<int64_t>(max_tiles_));
    vcnt_off_ = ap.alloc(4 * static_cast<int64_t>((n_ + dev::kVsChunk - 1) / dev::kVsChunk + 1) * plan_.k);
    ensure_tile_tot(max_tiles_);
  }
  if (need_rooted_) {
    const int slots = sched_.at(1)[0].nslots;
    for (auto& e : exec_)
      if (e.rooted) rooted_partial = std::max<int64_t>(rooted_partial, static_cast<int64_t>(slots) * static_cast<int64_t>(e.rooted_smem / (4 * dev::kSpmmWarps * (128 / e.rl_zw))));
  }
  // tables read by a pair expansion must be plain RR (not streamed-packed)
  std::vector<char> feeds_pair(plan_.num_nodes, 0);
  for (const auto& y : exec_)
    if (y.pair) feeds_pair[y.p] = 1;
  for (const auto& x : exec_)
    if (x.dup_of >= 0 && feeds_pair[x.id]) feeds_pair[exec_[x.dup_of].id] = 1;
  // Virtual active-leaf tables: an active-leaf node read only as its parent's
  // ACTIVE child is M_s[v, S] = P'[v, S minus c(v)], so the parent stages P'
  // through this node's per-color P' map and the permuted copy is never
  // written (TCG_VIRT=0 disables; inspection contexts materialize it).
  static const int virt_mode = [] {
    const char* s = std::getenv("TCG_VIRT");
    return s ? std::atoi(s) : 1;
  }();
  {
    std::vector<int> active_uses(plan_.num_nodes, 0), aliased(plan_.num_nodes, 0);
    for (const auto& y : exec_) {
      if (y.dup_of < 0 && !y.a_leaf) ++active_uses[y.a];
      if (y.dup_of >= 0) aliased[exec_[y.dup_of].id] = 1;
    }
    std::vector<char> pair_virt_ok(plan_.num_nodes, 0);  // a pair parent has the composed map
    for (const auto& y : exec_)
      if (y.pair && y.d_xmap_v && y.dup_of < 0) pair_virt_ok[y.p] = 1;
    for (auto& e : exec_) {
      // (a plan that streams active-leaf SpMMs to fit the device keeps streaming them)
      const bool base = virt_mode && !keep && !allow_stream && rooted_ema_ && e.a_leaf && !e.root && e.rooted &&
                        !e.p_leaf && e.dup_of < 0 && !aliased[e.id];
      // read only as an active child (staged through its P' map), or only by a
      // pair expansion (through the composed map)
      e.virt_px = base && feeds_pair[e.id] && pair_virt_ok[e.id] && active_uses[e.id] == 0;
      e.virt = (base && active_uses[e.id] == 1 && !feeds_pair[e.id]) || e.virt_px;
    }
  }
  for (auto& e : exec_) {
    if (e.dup_of >= 0) {  // alias the first occurrence; release this node's own children
      const NodeExec& x = exec_[e.dup_of];
      table_off_[e.id] = table_off_[x.id];
      e.out_off = x.out_off;
      e.pp_off = x.pp_off;
      if (!e.p_leaf) pprime_off_[e.p] = pprime_off_[x.p];
      // (the first occurrence's table was retained once per duplicate when
      // allocated; this node's parent releases that reference)
      if (!keep) {
        if (!e.p_leaf) ap.free(table_off_[e.p]);
        if (!e.a_leaf) ap.free(table_off_[e.a]);
      }
      continue;
    }
    e.pstream = false;
    if (allow_stream && rooted_ema_ && e.a_leaf && !e.root && e.rooted && !e.p_leaf && e.d_emap && e.pp_dup_of < 0 &&
        !feeds_pair[e.id] && !e.virt) {
      bool shared = false;
      for (const auto& y : exec_) shared |= y.pp_dup_of >= 0 && exec_[y.pp_dup_of].id == e.id;
      e.pstream = !shared;
    }
    if (e.pstream) {  // scratch for one group's P' columns + the output; M_p read meanwhile
      e.Ct = 0;
      for (int g = 0; g < e.rl_groups; ++g)
        e.Ct = std::max(e.Ct, (g + 1 < e.rl_groups ? e.rl_fbase[g + 1] : e.Cps) - e.rl_fbase[g]);
      e.pp_off = ap.alloc(table_bytes(e.Ct));
      pprime_off_[e.p] = -1;
      e.out_off = ap.alloc(table_bytes(e.Cout));
      table_off_[e.id] = e.out_off;
      for (const auto& y : exec_)
        if (y.dup_of >= 0 && exec_[y.dup_of].id == e.id) ap.retain(e.out_off);
      if (!keep) ap.free(table_off_[e.p]);
      ap.free(e.pp_off);
      continue;
    }
    if (e.pp_dup_of >= 0) {  // P' identical to an earlier node's: alias it
      e.pp_off = exec_[e.pp_dup_of].pp_off;
      pprime_off_[e.p] = e.pp_off;
      if (!keep) ap.free(table_off_[e.p]);
    } else if (!e.p_leaf && e.rooted && rooted_ema_ && e.pair) {
      // RR M_p expanded into its per-row-color copies, then dropped; P'
      // while the copies live
      e.ct_off = ap.alloc(4ll * plan_.k * e.rl_groups * e.rl_zw * n_);
      if (!keep) ap.free(table_off_[e.p]);
      e.pp_off = ap.alloc(table_bytes(e.Cps));
      pprime_off_[e.p] = e.pp_off;
      if (!keep) ap.free(e.ct_off);
    } else if (!e.p_leaf && e.rooted && rooted_ema_) {
      // M_p is already in the SpMM's compressed slot layout
      e.pp_off = ap.alloc(table_bytes(e.Cps));
      pprime_off_[e.p] = e.pp_off;
      if (!keep) ap.free(table_off_[e.p]);
    } else if (!e.p_leaf && e.rooted) {
      // compress M_p (alive), drop it, then P' while the compressed table lives
      e.ct_off = ap.alloc(table_bytes(static_cast<int64_t>(e.rl_groups) * e.rl_zw));
      if (!keep) ap.free(table_off_[e.p]);
      e.pp_off = ap.alloc(table_bytes(e.Cps));
      pprime_off_[e.p] = e.pp_off;
      if (!keep) ap.free(e.ct_off);
    } else if (!e.p_leaf) {
      e.pp_off = ap.alloc(table_bytes(e.Cp));
      pprime_off_[e.p] = e.pp_off;
      if (!keep) ap.free(table_off_[e.p]);
    }
    if (!e.p_leaf && e.pp_dup_of < 0)
      for (const auto& y : exec_)  // one reference per node sharing this P'
        if (y.pp_dup_of >= 0 && exec_[y.pp_dup_of].id == e.id) ap.retain(e.pp_off);
    if (e.virt) {  // the table IS P' (released by the parent, which reads it as its active child)
      table_off_[e.id] = e.out_off = e.pp_off;
      continue;
    }
    e.out_off = ap.alloc(e.root ? 8 * static_cast<int64_t>(n_) : table_bytes(rooted_ema_ ? e.Cout : e.Cs));
    table_off_[e.id] = e.out_off;
    for (const auto& y : exec_)  // one reference per duplicate's consumer
      if (y.dup_of >= 0 && exec_[y.dup_of].id == e.id) ap.retain(e.out_off);
    if (!keep) {
      if (!e.p_leaf) ap.free(e.pp_off);
      if (!e.a_leaf) ap.free(table_off_[e.a]);
    }
  }
  // consumers of a packed (streamed, RR) active table stage it through its amap
  for (auto& e : exec_) {
    e.d_amap_in = nullptr;
    e.Ca_in = e.Wa;
    if (e.a_leaf) continue;
    for (const auto& x : exec_)
      if (x.id == e.a) {
        const NodeExec& src = x.dup_of >= 0 ? exec_[x.dup_of] : x;
        if (src.pstream && src.omap.empty()) e.d_amap_in = src.d_amap;
        if (src.virt) {  // stage the child's P' through its P' map
          e.d_amap_in = src.d_pmap;
          e.Ca_in = src.Cpt;
        }
      }
  }
  // blocked rooted eMA with TMA-engine staging (opt-in, TCG_RT_TMA=1) when
  // the raw rows of a tile and its transposed buffers fit one SM.  Measured on
  // cfg3 node 1: 7.9 ms against 3.2 ms for the 2-CTA ema_rt_blocked -- one CTA
  // per SM leaves the per-tile group-queue tail exposed (55% of stalls at the
  // end-of-tile barrier: 26 output groups for 16 warps), and the raw buffer
  // leaves no room for a second CTA.
  static const int tma_mode = [] {
    const char* s = std::getenv("TCG_RT_TMA");
    return s ? std::atoi(s) : 0;
  }();
  // opt-in (TCG_RT_PIPE=1): the warp-specialized pipeline (two transposed
  // tiles per SM, producer warps staging with 4-byte cp.async, one group queue
  // across tiles) when two tiles fit and every tile has a group per consumer
  // warp.  Measured on cfg3 node 1 (producer/consumer warps -> ms): 1/16 7.4,
  // 2/16 4.9, 4/16 4.0, 8/12 3.45, 8/16 3.40, against 3.33-3.47 for the
  // 2-CTA ema_rt_blocked: the 4-byte transposing copies, not the compute,
  // bound it, so the simple kernel stays the default.
  static const int pipe_mode = [] {
    const char* s = std::getenv("TCG_RT_PIPE");
    return s ? std::atoi(s) : 0;
  }();
  for (auto& e : exec_) {
    e.rt_tma_smem = e.rt_pipe_smem = 0;
    if (!rooted_ema_ || !e.rt_blocked || e.rt_vtx || e.root || e.a_leaf) continue;
    if (tma_mode) {
      const int64_t RS = static_cast<int64_t>(dev::num_panels(e.Ca_in) + dev::num_panels(e.Cpt)) * dev::kZ;
      const int64_t sm = 4 * (32 * RS + static_cast<int64_t>(e.Wa + e.Wp) * dev::kSpitch);
      if (sm <= max_smem_ - 4096) e.rt_tma_smem = static_cast<size_t>(sm);
    } else if (pipe_mode && e.rt_ngroups >= dev::kRtPipeConsumers) {
      const int64_t sm = 4 * 2 * static_cast<int64_t>(e.Wa + e.Wp) * dev::kSpitch;
      if (sm <= max_smem_ - 4096) e.rt_pipe_smem = static_cast<size_t>(sm);
    }
  }
  arena_bytes_ = ap.peak;
  partial_bytes_ = std::max<int64_t>(static_cast<int64_t>(max_slots_) * dev::kZ * 8, rooted_partial * 8);
}

int64_t Engine::required_bytes() const {
  require_ready();
  int64_t sched = 0;
  for (auto& kv : sched_)
    for (auto& s : kv.second) sched += s.nseg_padded;
  const int64_t graph = 8 * (static_cast<int64_t>(n_) + 1) + 4 * nnz_ +
                        static_cast<int64_t>(sizeof(dev::Seg)) * sched;
  return arena_bytes_ + partial_bytes_ + graph + n_ + 8 * ((n_ + 31) / 32);
}

void Engine::require_ready() const {
  if (n_ < 0) throw invalid_argument("no graph set (tcg_set_graph)");
  if (!have_template_) throw invalid_argument("no template set (tcg_set_template)");
}

void Engine::ensure_arena() {
  require_ready();
  if (cfg_.memory_budget > 0 && arena_bytes_ > cfg_.memory_budget)
    throw resource_error("count tables need " + std::to_string(arena_bytes_) +
                         " bytes, over the budget of " + std::to_string(cfg_.memory_budget));
  if (arena_bytes_ > arena_alloc_ || !arena_) {  // (grow only: no free/malloc per graph)
    dfree(arena_);
    arena_alloc_ = 0;
    TCG_CUDA(cudaMalloc(&arena_, std::max<int64_t>(arena_bytes_, kAlign)));
    arena_alloc_ = arena_bytes_;
  }
  if (partial_bytes_ > partial_alloc_) {
    dfree(d_partial_);
    partial_alloc_ = 0;
    if (partial_bytes_) TCG_CUDA(cudaMalloc(&d_partial_, partial_bytes_));
    partial_alloc_ = partial_bytes_;
  }
}

void Engine::ensure_colors(int64_t bytes) {
  if (colors_cap_ < bytes) {
    dfree(d_colors_);
    colors_cap_ = 0;
    TCG_CUDA(cudaMalloc(&d_colors_, std::max<int64_t>(bytes, 1)));
    colors_cap_ = bytes;
  }
}

// ----------------------------------------------------------------- colors
void Engine::gen_colors(const uint64_t* seeds, int count, uint8_t* d_out) {
  TCG_CUDA(cudaMemcpyAsync(d_seeds_, seeds, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, stream_));
  const uint64_t k = static_cast<uint64_t>(plan_.k);
  const uint64_t limit = limit_override_ ? limit_override_ : (UINT64_MAX / k) * k;
  // every rank generates the full (global) coloring: the MT stream is serial
  dev::mt_coloring<<<count, dev::kMtThreads, 0, stream_>>>(d_seeds_, nglob_, plan_.k, limit, UINT64_MAX / k,
                                                             d_out, nglob_);
  ++launches_;
  TCG_CUDA(cudaGetLastError());
}

// The coloring of `seed`: the prefetched one when it matches this graph, template and rejection
// limit (the DP then waits for the side stream's event), else generated on the engine stream.
const uint8_t* Engine::take_or_generate(uint64_t seed) {
  const uint64_t k = static_cast<uint64_t>(plan_.k);
  const uint64_t limit = limit_override_ ? limit_override_ : (UINT64_MAX / k) * k;
  if (next_.valid && next_.seed == seed && next_.n == nglob_ && next_.k == plan_.k && next_.limit == limit) {
    next_.valid = false;
    TCG_CUDA(cudaStreamWaitEvent(stream_, next_.ready, 0));
    return next_.d_buf[next_.cur];
  }
  gen_colors(&seed, 1, d_colors_);
  return d_colors_;
}

// Generate the coloring of `seed` on the side stream into the buffer the running DP does not read.
void Engine::prefetch_next(uint64_t seed) {
  // (small graphs: the generation is tens of microseconds, less than a second launch is worth)
  if (nglob_ < (1 << 16) || exec_.empty()) return;
  if (!next_.stream) {
    TCG_CUDA(cudaStreamCreateWithFlags(&next_.stream, cudaStreamNonBlocking));
    TCG_CUDA(cudaEventCreateWithFlags(&next_.ready, cudaEventDisableTiming));
    TCG_CUDA(cudaMalloc(&next_.d_seed, sizeof(uint64_t)));
  }
  if (next_.cap < nglob_) {
    TCG_CUDA(cudaStreamSynchronize(next_.stream));
    for (auto& b : next_.d_buf) {
      dfree(b);
      TCG_CUDA(cudaMalloc(&b, nglob_));
    }
    next_.cap = nglob_;
  }
  const uint64_t k = static_cast<uint64_t>(plan_.k);
  const uint64_t limit = limit_override_ ? limit_override_ : (UINT64_MAX / k) * k;
  next_.cur ^= 1;
  TCG_CUDA(cudaMemcpyAsync(next_.d_seed, &seed, sizeof(uint64_t), cudaMemcpyHostToDevice, next_.stream));
  dev::mt_coloring<<<1, dev::kMtThreads, 0, next_.stream>>>(next_.d_seed, nglob_, plan_.k, limit, UINT64_MAX / k,
                                                           next_.d_buf[next_.cur], nglob_);
  ++launches_;
  TCG_CUDA(cudaGetLastError());
  TCG_CUDA(cudaEventRecord(next_.ready, next_.stream));
  next_.valid = true;
  next_.seed = seed;
  next_.limit = limit;
  next_.n = nglob_;
  next_.k = plan_.k;
}

void Engine::coloring(uint64_t seed, uint8_t* host_colors) {
  require_ready();
  TCG_CUDA(cudaSetDevice(cfg_.device));
  ensure_colors(nglob_);
  gen_colors(&seed, 1, d_colors_);
  TCG_CUDA(cudaMemcpyAsync(host_colors, d_colors_, nglob_, cudaMemcpyDeviceToHost, stream_));
  TCG_CUDA(cudaStreamSynchronize(stream_));
}

// colors in padded-global order (the gather ids of a sharded graph)
void Engine::gather_colors(const uint8_t* d_colors) {
  const int64_t nmax = n_;
  dev::pad_colors<<<static_cast<unsigned>((nsrc_ + 255) / 256), 256, 0, stream_>>>(d_colors, d_rows_, nmax, nsrc_,
                                                                                   d_colors_pad_);
  ++launches_;
  TCG_CUDA(cudaGetLastError());
}

// rooted totals of `count` colorings: all-gather the per-rank fp64 partials
// and sum them in rank order (deterministic)
void Engine::finish_shard_totals(double* totals, int count) {
  if (!sharded()) return;
  static const bool dbg = std::getenv("TCG_DEBUG_SHARD") != nullptr;
  if (dbg)
    std::fprintf(stderr, "[tcg shard %d/%d] rows [%lld,%lld) nmax %d nsrc %d local total[0] %.6e\n", rank_,
                 world_, static_cast<long long>(rows_[rank_]), static_cast<long long>(rows_[rank_ + 1]), n_,
                 nsrc_, totals[0]);
  std::vector<double> all(static_cast<size_t>(count) * world_);
  for (int i0 = 0; i0 < count; i0 += 2048) {
    const int c = std::min(2048, count - i0);
    TCG_CUDA(cudaMemcpyAsync(d_gather_, totals + i0, sizeof(double) * c, cudaMemcpyHostToDevice, stream_));
    tr_->allgather(d_gather_, sizeof(double) * c, d_gather_ + 2048, stream_);
    std::vector<double> part(static_cast<size_t>(c) * world_);
    TCG_CUDA(cudaMemcpyAsync(part.data(), d_gather_ + 2048, sizeof(double) * c * world_, cudaMemcpyDeviceToHost, stream_));
    TCG_CUDA(cudaStreamSynchronize(stream_));
    if (dbg && i0 == 0)
      for (int r = 0; r < world_; ++r)
        std::fprintf(stderr, "[tcg shard %d/%d] gathered[%d] %.6e\n", rank_, world_, r, part[static_cast<size_t>(r) * c]);
    for (int j = 0; j < c; ++j) {
      double s = 0.0;
      for (int r = 0; r < world_; ++r) s += part[static_cast<size_t>(r) * c + j];
      totals[i0 + j] = s;
    }
  }
}

void Engine::copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  TCG_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, stream_));
  TCG_CUDA(cudaStreamSynchronize(stream_));
}

// per-vertex fp64 values of the local rows -> global vector on the host
void Engine::gather_per_vertex(const double* d_local, double* host_global) {
  double* d_all = nullptr;
  TCG_CUDA(cudaMalloc(&d_all, sizeof(double) * static_cast<size_t>(n_) * world_));
  std::vector<double> all(static_cast<size_t>(n_) * world_);
  try {
    tr_->allgather(d_local, sizeof(double) * n_, d_all, stream_);
    TCG_CUDA(cudaMemcpyAsync(all.data(), d_all, all.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    TCG_CUDA(cudaStreamSynchronize(stream_));
  } catch (...) {
    cudaFree(d_all);
    throw;
  }
  cudaFree(d_all);
  for (int r = 0; r < world_; ++r)
    for (int64_t j = 0; j < rows_[r + 1] - rows_[r]; ++j)
      host_global[rows_[r] + j] = all[static_cast<size_t>(r) * n_ + j];
}

// ------------------------------------------------------------------- SpMM
template <int ZW, bool ONEHOT>
static void launch_spmm_part(const PartSchedule& ps, cudaStream_t s, const int32_t* col,
                             const float* X, const uint8_t* colors, int color_base, float* Y,
                             double* partial, bool first, int64_t& launches) {
  constexpr int spw = 128 / ZW;  // segments per warp
  const int64_t ntasks = ps.nseg_padded / spw;
  const int64_t blocks = (ntasks + dev::kSpmmWarps - 1) / dev::kSpmmWarps;
  dev::spmm_part<ZW, ONEHOT><<<static_cast<unsigned>(blocks), dev::kSpmmWarps * 32, 0, s>>>(
      ps.d_segs, ntasks, col, X, colors, color_base, Y, partial, first ? 1 : 0);
  ++launches;
  if (ps.nsplit_rows) {
    const int64_t total = static_cast<int64_t>(ps.nsplit_rows) * ZW;
    dev::spmm_fixup<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
        ps.d_split_rows, ps.d_slot_begin, ps.nsplit_rows, partial, Y, ZW, first ? 1 : 0);
    ++launches;
  }
}

void Engine::spmm(const float* X, float* Y, int64_t cols) {
  const int P = dev::num_panels(cols);
  for (int p = 0; p < P; ++p) {
    const int zw = dev::panel_width(cols, p);
    const float* Xp = X + static_cast<int64_t>(p) * n_ * dev::kZ;
    float* Yp = Y + static_cast<int64_t>(p) * n_ * dev::kZ;
    if (sharded()) {
      // the gather source is every rank's panel: all-gather it (rank blocks
      // of nmax rows = the padded-global ids of the local CSR)
      tr_->allgather(Xp, sizeof(float) * static_cast<size_t>(n_) * zw, d_xfull_, stream_);
      Xp = d_xfull_;
    }
    const auto& parts = sched_.at(parts_for_width(zw));
    const int P = static_cast<int>(parts.size());
    for (int s = 0; s < P; ++s) {
      const PartSchedule& ps = parts[s];
      if (zw == 32) launch_spmm_part<32, false>(ps, stream_, d_col_, Xp, nullptr, 0, Yp, d_partial_, s == 0, launches_);
      else if (zw == 16) launch_spmm_part<16, false>(ps, stream_, d_col_, Xp, nullptr, 0, Yp, d_partial_, s == 0, launches_);
      else launch_spmm_part<8, false>(ps, stream_, d_col_, Xp, nullptr, 0, Yp, d_partial_, s == 0, launches_);
    }
  }
  TCG_CUDA(cudaGetLastError());
}

// Rooted-color compressed SpMM (host.hpp RootedLayout, kernels.cuh): compress
// M_p to its color-rooted slots, then one pass per (group, part) over the
// (part, color)-sorted rows, each producing the group's P' columns.
void Engine::rooted_spmm(const NodeExec& e, const float* M, float* Pp, const uint8_t* d_colors, float* out) {
  const int k = e.slot_K + (e.pair ? 1 : 0);
  const int zw = e.rl_zw, G = e.rl_groups;
  const float* X = rooted_ema_ ? M : table_ptr(e.ct_off);
  int64_t xstride = 0;  // pair layout: floats between the copies of two row colors
  if (e.pair) {
    if (sharded()) throw logic_error("pair-layout SpMM on a sharded context");
    float* cp = table_ptr(e.ct_off);
    // a virtual active-leaf child: its P' (storage columns) through the composed map
    const NodeExec* ch = nullptr;
    for (const auto& x : exec_)
      if (x.id == e.p) ch = &x;
    const bool vpx = ch && ch->virt_px;
    const int wx = vpx ? ch->Cpt : e.Wx;
    const size_t smem = static_cast<size_t>(4) * 32 * (wx + 1);
    smem_limit(reinterpret_cast<const void*>(dev::pair_expand), smem);
    dev::pair_expand<<<static_cast<unsigned>((n_ + 31) / 32), 256, smem, stream_>>>(M, wx, d_colors, vpx ? e.d_xmap_v : e.d_xmap,
                                                                                      k, G, zw, n_, cp);
    ++launches_;
    X = cp;
    xstride = static_cast<int64_t>(G) * n_ * zw;
  }
  if (!rooted_ema_) {
    const int rf = static_cast<int>(dev::table_floats(e.Cp, 1));
    const int vpb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(32, (96 << 10) / (4 * rf))));
    const size_t smem = static_cast<size_t>(vpb) * rf * 4;
    smem_limit(reinterpret_cast<const void*>(dev::rooted_compress), smem);
    dev::rooted_compress<<<static_cast<unsigned>((n_ + vpb - 1) / vpb), 256, smem, stream_>>>(
        M, e.Cp, d_colors, e.d_slot_col, G, zw, n_, vpb, table_ptr(e.ct_off));
    ++launches_;
  }
  const PartSchedule& ps = sched_.at(1)[0];  // whole rows; parts = color classes
  const uint32_t* colb = reinterpret_cast<const uint32_t*>(arena_ + rcol_off_);
  const int64_t* cuts = reinterpret_cast<const int64_t*>(arena_ + rcut_off_);
  // (4 CTAs per SM at 64 registers: the occupancy sweep in DESIGN.md 3)
  auto pick = [&](auto pair_tag) -> const void* {
    constexpr bool P = decltype(pair_tag)::value;
    return zw == 32 ? reinterpret_cast<const void*>(dev::spmm_rooted<32, 4, P>)
           : zw == 16 ? reinterpret_cast<const void*>(dev::spmm_rooted<16, 4, P>)
                      : reinterpret_cast<const void*>(dev::spmm_rooted<8, 4, P>);
  };
  const void* kern = e.pair ? pick(std::true_type{}) : pick(std::false_type{});
  // pair: the rows in color order (this coloring's re-ordered schedule)
  const dev::Seg* segs = e.pair ? reinterpret_cast<const dev::Seg*>(arena_ + pseg_off_) : ps.d_segs;
  const uint8_t* rowc = e.pair ? d_colors : nullptr;
  smem_limit(reinterpret_cast<const void*>(kern), e.rooted_smem);
  const int spw = 128 / zw;
  // sharded + async transport (NCCL): group g+1's panel is all-gathered on the
  // communication stream while group g's SpMM runs (two buffers; event
  // ordering only, no host synchronization)
  const bool pipe = sharded() && tr_->async();
  float* xbuf[2] = {d_xfull_, d_xfull2_};
  auto gather_async = [&](int g) {
    const float* src = X + static_cast<int64_t>(g) * n_ * (e.pair ? zw : dev::kZ);
    if (g >= 2) TCG_CUDA(cudaStreamWaitEvent(comm_, ev_u_[g % 2], 0));  // SpMM g-2 done reading the buffer
    tr_->allgather(src, sizeof(float) * static_cast<size_t>(n_) * zw, xbuf[g % 2], comm_);
    TCG_CUDA(cudaEventRecord(ev_g_[g % 2], comm_));
  };
  if (pipe && G > 0) {
    TCG_CUDA(cudaEventRecord(ev_in_, stream_));  // the passive table is complete
    TCG_CUDA(cudaStreamWaitEvent(comm_, ev_in_, 0));
    gather_async(0);
  }
  for (int g = 0; g < G; ++g) {
    const float* Xg = X + static_cast<int64_t>(g) * n_ * (e.pair ? zw : dev::kZ);
    if (pipe) {
      if (g + 1 < G) gather_async(g + 1);
      TCG_CUDA(cudaStreamWaitEvent(stream_, ev_g_[g % 2], 0));
      Xg = xbuf[g % 2];
    } else if (sharded()) {
      tr_->allgather(Xg, sizeof(float) * static_cast<size_t>(n_) * zw, d_xfull_, stream_);
      Xg = d_xfull_;
    }
    const int gbase = e.rl_fbase[g];
    const int fpad = (g + 1 < G ? e.rl_fbase[g + 1] : e.Cps) - gbase;
    const int fbase = out ? 0 : gbase;       // streamed: the group's columns at 0 of the scratch
    const int32_t Cst = out ? e.Ct : e.Cps;
    const size_t smem = static_cast<size_t>(dev::kSpmmWarps) * spw * (fpad + 4) * 4 + 2 * (e.slot_K + 1) * zw;
    const int16_t* sl = e.d_slot_acc + static_cast<int64_t>(g) * zw;
    int slot_stride = G * zw;
    for (int q = 0; q < rooted_parts_; ++q) {
      const int64_t ntasks = ps.nseg_padded / spw;
      const unsigned blocks = static_cast<unsigned>((ntasks + dev::kSpmmWarps - 1) / dev::kSpmmWarps);
      const int first = q == 0 ? 1 : 0;
      int part = q;
      void* args[] = {const_cast<dev::Seg**>(&segs), const_cast<int64_t*>(&ntasks), const_cast<uint32_t**>(&colb),
                      const_cast<int64_t**>(&cuts), &rooted_parts_, &part, const_cast<int32_t**>(&ps.d_slot_row),
                      const_cast<float**>(&Xg), const_cast<int16_t**>(&sl), &slot_stride, const_cast<int*>(&fbase),
                      const_cast<int*>(&fpad), const_cast<int32_t*>(&Cst), &n_, &Pp, &d_partial_,
                      const_cast<int*>(&first), const_cast<uint8_t**>(&rowc), &xstride, const_cast<int*>(&e.slot_K)};
      TCG_CUDA(cudaLaunchKernel(kern, dim3(blocks), dim3(dev::kSpmmWarps * 32), args, smem, stream_));
      ++launches_;
      if (ps.nsplit_rows) {
        const int64_t total = static_cast<int64_t>(ps.nsplit_rows) * fpad;
        dev::rooted_fixup<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream_>>>(
            ps.d_split_rows, ps.d_slot_begin, ps.nsplit_rows, d_partial_, fbase, fpad, Cst, n_, Pp, first);
        ++launches_;
      }
    }
    if (pipe) TCG_CUDA(cudaEventRecord(ev_u_[g % 2], stream_));
    if (out) {  // the group's P' columns are complete: scatter into the active-leaf output
      const int64_t total = static_cast<int64_t>(n_) * fpad;
      dev::pstream_copy<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 64)), 256, 0, stream_>>>(
          Pp, e.Ct, fpad, e.d_emap + gbase, e.Cps, d_colors, e.Cout, n_, out);
      ++launches_;
    }
  }
  TCG_CUDA(cudaGetLastError());
}

// P' of a leaf passive child: SpMM against the one-hot color table, read as
// 1-byte colors (whole rows; the colors array is L2-resident).
int Engine::parts_for_width(int zw) const {
  const int64_t need = (static_cast<int64_t>(nsrc_) * zw * 4 + part_bytes_ - 1) / part_bytes_;
  int P = 1;
  while (P < need && P < (1 << 20)) P *= 2;
  return std::max(1, std::min<int>(P, std::max(1, nsrc_)));
}

void Engine::hist(const uint8_t* d_colors, float* H) {
  const PartSchedule& full_ = sched_.at(1)[0];
  const int zw = dev::panel_width(plan_.k, 0);
  if (zw == 32) launch_spmm_part<32, true>(full_, stream_, d_col_, nullptr, d_colors, 0, H, d_partial_, true, launches_);
  else if (zw == 16) launch_spmm_part<16, true>(full_, stream_, d_col_, nullptr, d_colors, 0, H, d_partial_, true, launches_);
  else launch_spmm_part<8, true>(full_, stream_, d_col_, nullptr, d_colors, 0, H, d_partial_, true, launches_);
  TCG_CUDA(cudaGetLastError());
}

// -------------------------------------------------------------------- eMA
template <bool AL, bool ST>
static void launch_node(const NodeExec& e, int k, cudaStream_t s, int32_t n, const float* A,
                        const float* P, const uint8_t* colors, float* out) {
  auto kern = dev::ema_node<AL, ST>;
  smem_limit(reinterpret_cast<const void*>(kern), e.ema_smem);
  const unsigned tiles = static_cast<unsigned>((n + dev::kTileV - 1) / dev::kTileV);
  // one warp per 8-column output chunk (up to 16): light nodes get small CTAs,
  // so many tiles co-reside per SM and staging overlaps compute across CTAs
  const int warps = std::max(2, std::min(dev::kEmaWarps, (e.Cs + 7) / 8));
  kern<<<tiles, warps * 32, e.ema_smem, s>>>(A, P, colors, e.d_split, e.d_packed, e.d_drop, k,
                                             e.pairs, e.Ca, e.Cps, e.Cs, n, out);
}

template <bool AL, bool ST>
static void launch_root(const NodeExec& e, cudaStream_t s, int32_t n, const float* A,
                        const float* P, const uint8_t* colors, double* rout, double* racc,
                        double* tile_tot) {
  auto kern = dev::ema_root<AL, ST>;
  smem_limit(reinterpret_cast<const void*>(kern), e.ema_smem);
  const unsigned tiles = static_cast<unsigned>((n + dev::kTileV - 1) / dev::kTileV);
  kern<<<tiles, dev::kEmaWarps * 32, e.ema_smem, s>>>(A, P, colors, e.d_split, e.pairs, e.Ca, e.Cps,
                                                      n, rout, racc, tile_tot);
}

// Rooted eMA of one node over the same-color tiles (kernels_rt.cuh).
void Engine::launch_rt_ema(const NodeExec& e, const float* A, const float* P, double* d_root_acc) {
  const int32_t* vs = reinterpret_cast<const int32_t*>(arena_ + vs_off_);
  const int4* tl = reinterpret_cast<const int4*>(arena_ + tiles_off_);
  const unsigned grid = static_cast<unsigned>(max_tiles_);
  auto attr = [&](const void* f) {
    smem_limit(f, e.rt_smem);
  };
  if (e.rtv_pleaf) {  // vertex-per-warp over a leaf passive child
    const int slice = (e.Wa + 31) / 32 * 32 + 32 + 1;  // (+1: vertices' rows on different banks)
    const int cst = e.omap.empty() ? e.Ws : e.Cout;
    const int oslice = (cst + 31) / 32 * 32 + 1;
    // one vertex per CTA pass (measured cfg4 node 4 / node 7, V = 1 / 2 / 4: 44 / 48 / 68 and 12.5 / 11.2 / 10.4 ms)
    const size_t smem = static_cast<size_t>(slice + oslice) * 4;
    using PleafFn = void (*)(const float*, int, const int32_t*, int, const float*, int, const int32_t*, const uint8_t*,
                             const uint32_t*, int, int, const int32_t*, int, int32_t, int, int, float*);
    static const PleafFn kerns[7] = {dev::ema_rtv_pleaf<1, 0>, dev::ema_rtv_pleaf<1, 1>, dev::ema_rtv_pleaf<1, 2>,
                                     dev::ema_rtv_pleaf<1, 3>, dev::ema_rtv_pleaf<1, 4>, dev::ema_rtv_pleaf<1, 5>,
                                     dev::ema_rtv_pleaf<1, 6>};
    const PleafFn kern = kerns[e.rtv_packed ? e.size - 1 : 0];
    smem_limit(reinterpret_cast<const void*>(kern), smem);
    const unsigned pgrid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(n_, 148 * 16)));
    kern<<<pgrid, 256, smem, stream_>>>(A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, d_colors_rt_, e.d_rtv_drop, e.size - 1,
                                        e.Ws, e.d_omap, e.Cout, n_, slice, oslice, table_ptr(e.out_off));
    return;
  }
  if (e.rt_vtx) {
    const unsigned vgrid = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>((n_ + e.rtv_V - 1) / e.rtv_V, e.root ? 148 * 16 : 148 * 2 * 8)));
    if (e.root) {
      double* rout = reinterpret_cast<double*>(arena_ + e.out_off);
      attr(reinterpret_cast<const void*>(dev::ema_rtv_root));
      dev::ema_rtv_root<<<vgrid, 256, e.rt_smem, stream_>>>(A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, d_colors_rt_, e.d_rt_split,
                                                             e.rt_pairs, n_, rout, d_root_acc);
    } else {
      // two CTAs of 14 warps per SM (72 registers, no spills).  Measured on cfg5 node 1 / node 2,
      // threads per CTA 256 / 320 / 384 / 448 / 512: 238 / 232 / 230 / 217 / 230 and 111 / 103 / 102 /
      // 100 / 101 ms (512: 64 registers, spills); three 256-thread CTAs when V allows: cfg4 node 1
      // 103 against 102 ms
      const int thr = e.rtv_one_cta ? 2 * dev::kRtvThreads : dev::kRtvThreads;
      auto kern = e.rtv_one_cta ? dev::ema_rtv_blocked<dev::kH1, 2 * dev::kRtvThreads>
                                : dev::ema_rtv_blocked<dev::kH1, dev::kRtvThreads>;
      attr(reinterpret_cast<const void*>(kern));
      kern<<<vgrid, thr, e.rt_smem, stream_>>>(
          A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, d_colors_rt_, static_cast<const dev::RtvTask*>(e.d_rtv_tasks), e.rtv_ntasks, e.d_rtv_gout,
          e.d_rtv_runs, e.d_rtv_blocks, e.Ws, e.d_omap, e.Cout, n_, table_ptr(e.out_off), e.rtv_V, e.rtv_sa, e.rtv_sp);
    }
    return;
  }
  if (e.root) {
    double* rout = reinterpret_cast<double*>(arena_ + e.out_off);
    const int rwarps = std::max(2, std::min(dev::kEmaWarps, e.rt_pairs / 4));  // warps split the pairs
    if (e.a_leaf) {
      attr(reinterpret_cast<const void*>(dev::ema_rt_root<true>));
      dev::ema_rt_root<true><<<grid, 64, e.rt_smem, stream_>>>(
          A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, e.Wp, vs, tl, e.d_rt_split, e.rt_pairs, n_, rout, d_root_acc, d_tile_tot_);
    } else {
      attr(reinterpret_cast<const void*>(dev::ema_rt_root<false>));
      dev::ema_rt_root<false><<<grid, rwarps * 32, e.rt_smem, stream_>>>(
          A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, e.Wp, vs, tl, e.d_rt_split, e.rt_pairs, n_, rout, d_root_acc, d_tile_tot_);
    }
    return;
  }
  float* out = table_ptr(e.out_off);
  const int warps = std::max(2, std::min(dev::kEmaWarps, (e.Ws + 7) / 8));
  if (e.a_leaf) {
    const int rf = static_cast<int>(dev::table_floats(e.Cpt, 1));
    // (narrow rows: up to 128 vertices per CTA, so a CTA moves >= 16 KB)
    const int vpb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(128, (48 << 10) / (4 * rf))));
    const size_t smem = static_cast<size_t>(vpb) * rf * 4;
    smem_limit(reinterpret_cast<const void*>(dev::ema_rt_copy), smem);
    int L = 1;  // lanes per row: enough for the row's float4s and the output panel's slots
    while (L < 32 && (L * 4 < rf || L < std::min(32, e.Cout))) L *= 2;
    dev::ema_rt_copy<<<static_cast<unsigned>((n_ + vpb - 1) / vpb), 256, smem, stream_>>>(
        P, e.Cpt, d_colors_rt_, e.d_cmap, e.Cout, n_, vpb, L, out);
  } else if (e.rt_blocked && e.rt_pipe_smem) {
    auto kern = dev::ema_rt_blocked_pipe<dev::kRtPipeProducers, dev::kRtPipeConsumers>;
    const int nthr = (dev::kRtPipeProducers + dev::kRtPipeConsumers) * 32;
    smem_limit(reinterpret_cast<const void*>(kern), e.rt_pipe_smem);
    const unsigned g = static_cast<unsigned>(std::max(1, std::min(max_tiles_, num_sms_)));
    kern<<<g, nthr, e.rt_pipe_smem, stream_>>>(
        A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, e.Wp, vs, tl, max_tiles_,
        static_cast<const dev::GroupDesc*>(e.d_rt_groups), e.rt_ngroups, static_cast<const dev::BlockDesc*>(e.d_rt_blocks),
        e.Ws, e.d_omap, e.Cout, n_, out);
  } else if (e.rt_blocked && e.rt_tma_smem) {
    // persistent, TMA-engine staging double-buffered against the compute
    auto kern = dev::ema_rt_blocked_tma;
    smem_limit(reinterpret_cast<const void*>(kern), e.rt_tma_smem);
    const int RA = dev::num_panels(e.Ca_in) * dev::kZ;
    const int RS = RA + dev::num_panels(e.Cpt) * dev::kZ;
    const unsigned g = static_cast<unsigned>(std::max(1, std::min(max_tiles_, num_sms_)));
    kern<<<g, dev::kRtTmaThreads, e.rt_tma_smem, stream_>>>(
        A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, e.Wp, vs, tl, max_tiles_,
        static_cast<const dev::GroupDesc*>(e.d_rt_groups), e.rt_ngroups, static_cast<const dev::BlockDesc*>(e.d_rt_blocks),
        e.Ws, e.d_omap, e.Cout, n_, out, RS, RA);
  } else if (e.rt_blocked) {
    attr(reinterpret_cast<const void*>(dev::ema_rt_blocked));
    dev::ema_rt_blocked<<<grid, dev::kRtBlockedThreads, e.rt_smem, stream_>>>(
        A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, e.Wp, vs, tl, static_cast<const dev::GroupDesc*>(e.d_rt_groups), e.rt_ngroups,
        static_cast<const dev::BlockDesc*>(e.d_rt_blocks), e.Ws, e.d_omap, e.Cout, n_, out);
  } else {
    // narrow nodes: one warp per tile (8 tiles per CTA in flight) when a
    // warp's slice of A, P (and the staged RS output) is small
    static const int warp_mode = [] {
      const char* s = std::getenv("TCG_RT_WARP");
      return s ? std::atoi(s) : 1;
    }();
    const int slice = (e.Wa + e.Wp + (e.d_imap ? e.Ws : 0)) * dev::kSpitch;
    const size_t wsmem = static_cast<size_t>(8) * slice * 4;
    if (warp_mode && wsmem <= (100u << 10)) {
      smem_limit(reinterpret_cast<const void*>(dev::ema_rt_node_w), wsmem);
      dev::ema_rt_node_w<<<static_cast<unsigned>((max_tiles_ + 7) / 8), 256, wsmem, stream_>>>(
          A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, e.Wp, vs, tl, max_tiles_, e.d_rt_packed, e.rt_pairs, e.Ws,
          e.d_omap, e.d_imap, e.Cout, n_, slice, out);
      return;
    }
    attr(reinterpret_cast<const void*>(dev::ema_rt_node<false>));
    dev::ema_rt_node<false><<<grid, warps * 32, e.rt_smem, stream_>>>(
        A, e.Wa, e.d_amap_in, e.Ca_in, P, e.Cpt, e.d_pmap, e.Wp, vs, tl, e.d_rt_packed, e.rt_pairs, e.Ws, e.d_omap, e.d_imap, e.Cout, n_, out);
  }
}

// Per coloring: every row stably sorted by neighbour colour (rotated order,
// packed entries, part cuts) for the rooted SpMMs, the neighbour colour
// histogram hf (nullable) as a by-product, and -- for pair-layout SpMMs --
// the whole-row segments re-ordered by row colour.
void Engine::bucket_coloring(const uint8_t* d_gcolors, const uint8_t* d_colors, int k, float* hf, bool pair) {
  TCG_CUDA(cudaMemsetAsync(d_counter_, 0, sizeof(int), stream_));
  const size_t smem = sizeof(int) * 8 * k;
  uint32_t* rc = reinterpret_cast<uint32_t*>(arena_ + rcol_off_);
  int64_t* cuts = reinterpret_cast<int64_t*>(arena_ + rcut_off_);
  const int hzw = dev::panel_width(k, 0);
  if (nlong_ > 0) {  // hub rows: chunked over many CTAs
    int* ccnt = reinterpret_cast<int*>(arena_ + lcnt_off_);
    dev::bucket_long_count<<<static_cast<unsigned>(nlchunks_), 256, 0, stream_>>>(d_lchunks_, d_row_ptr_, d_col_, d_gcolors,
                                                                                   d_colors, k, ccnt);
    dev::bucket_long_scan<<<static_cast<unsigned>((nlong_ + 7) / 8), 256, 0, stream_>>>(
        d_lchunks_, d_lfirst_, d_row_ptr_, d_colors, nlong_, k, rooted_parts_, ccnt, cuts, hf, hzw);
    dev::bucket_long_scatter<<<static_cast<unsigned>(nlchunks_), 256, 0, stream_>>>(d_lchunks_, d_row_ptr_, d_col_, d_gcolors,
                                                                                     d_colors, k, ccnt, rc);
    launches_ += 3;
  }
  dev::bucket_rows<<<148 * 8, 256, smem, stream_>>>(d_row_ptr_, d_col_, d_gcolors, d_colors, d_row_order_, nlong_, nsmall_,
                                                   k, rooted_parts_, rc, cuts, hf, hzw);
  ++launches_;
  if (nsmall_ < n_) {
    dev::bucket_small<<<static_cast<unsigned>((n_ - nsmall_ + 255) / 256), 256, 0, stream_>>>(
        d_row_ptr_, d_col_, d_gcolors, d_colors, d_row_order_, nsmall_, n_, k, rooted_parts_, rc, cuts, hf, hzw);
    ++launches_;
  }
  if (pair) {  // whole-row segments re-ordered by row color (stable)
    const PartSchedule& ps = sched_.at(1)[0];
    const int64_t nseg = ps.nseg_padded;
    const int nchunks = static_cast<int>((nseg + dev::kVsChunk - 1) / dev::kVsChunk);
    uint8_t* keys = reinterpret_cast<uint8_t*>(arena_ + pkey_off_);
    int* pcnt = reinterpret_cast<int*>(arena_ + pcnt_off_);
    int32_t* perm = reinterpret_cast<int32_t*>(arena_ + pperm_off_);
    dev::seg_keys<<<static_cast<unsigned>((nseg + 255) / 256), 256, 0, stream_>>>(ps.d_segs, nseg, ps.d_slot_row, d_colors,
                                                                                 k, keys);
    dev::vsort_count<<<nchunks, 256, 0, stream_>>>(keys, static_cast<int32_t>(nseg), k + 1, pcnt);
    dev::vsort_scan<<<1, 1024, 0, stream_>>>(pcnt, nchunks, k + 1, nullptr, 0);
    dev::vsort_scatter<<<nchunks, 256, 0, stream_>>>(keys, static_cast<int32_t>(nseg), k + 1, pcnt, perm);
    dev::seg_gather<<<static_cast<unsigned>((nseg + 255) / 256), 256, 0, stream_>>>(
        ps.d_segs, perm, nseg, reinterpret_cast<dev::Seg*>(arena_ + pseg_off_));
    launches_ += 5;
  }
  TCG_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------- one DP
void Engine::run_dp(const uint8_t* d_colors_in, double* d_total, double* d_root_acc,
                    tcg_node_stats* stats) {
  if (relabeled_ && n_ > 0) {  // the caller's vertex order -> internal rows
    if (colors_rl_cap_ < n_) {
      dfree(d_colors_rl_);
      colors_rl_cap_ = 0;
      TCG_CUDA(cudaMalloc(&d_colors_rl_, n_));
      colors_rl_cap_ = n_;
    }
    dev::permute_colors<<<static_cast<unsigned>((n_ + 255) / 256), 256, 0, stream_>>>(d_colors_in, d_perm_, n_, d_colors_rl_);
    ++launches_;
    d_colors_in = d_colors_rl_;
  }
  // d_colors: colors of this context's rows (eMA); d_gcolors: by gather id
  const uint8_t* d_colors = d_colors_in;
  const uint8_t* d_gcolors = d_colors_in;
  if (sharded()) {
    gather_colors(d_colors_in);
    d_gcolors = d_colors_pad_;
    d_colors = d_colors_pad_ + static_cast<int64_t>(rank_) * n_;
  }
  std::vector<cudaEvent_t> ev;
  auto mark = [&]() {
    cudaEvent_t e;
    TCG_CUDA(cudaEventCreate(&e));
    TCG_CUDA(cudaEventRecord(e, stream_));
    ev.push_back(e);
    return ev.size() - 1;
  };
  const float* H = nullptr;
  if (need_hist_ && n_ > 0) {
    size_t h0 = 0;
    if (prof_) { h0 = prof_->used; TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
    if (!need_rooted_) {  // (with the rooted SpMM, bucket_rows writes it)
      hist(d_gcolors, table_ptr(hist_off_));
    }
    if (prof_) { prof_->spmm.emplace_back(h0, prof_->used); TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
    if (need_hist_) H = table_ptr(hist_off_);
  }
  if (need_rooted_ && n_ > 0) {
    // (part, color)-sorted packed rows for the rooted SpMMs of this coloring
    size_t b0 = 0;
    if (prof_) { b0 = prof_->used; TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
    // the bucketing counts ARE the neighbour color histogram: fused
    bucket_coloring(d_gcolors, d_colors, plan_.k, need_hist_ ? table_ptr(hist_off_) : nullptr, need_pair_);
    TCG_CUDA(cudaGetLastError());
    if (prof_) { prof_->spmm.emplace_back(b0, prof_->used); TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
  }
  d_colors_rt_ = d_colors;
  if (rooted_ema_ && n_ > 0) {
    // vertices sorted by color into same-color tiles for the rooted eMA
    size_t b0 = 0;
    if (prof_) { b0 = prof_->used; TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
    const int nchunks = static_cast<int>((n_ + dev::kVsChunk - 1) / dev::kVsChunk);
    int* vcnt = reinterpret_cast<int*>(arena_ + vcnt_off_);
    dev::vsort_count<<<nchunks, 256, 0, stream_>>>(d_colors, n_, plan_.k, vcnt);
    dev::vsort_scan<<<1, 1024, 0, stream_>>>(vcnt, nchunks, plan_.k, reinterpret_cast<int4*>(arena_ + tiles_off_), max_tiles_);
    dev::vsort_scatter<<<nchunks, 256, 0, stream_>>>(d_colors, n_, plan_.k, vcnt, reinterpret_cast<int32_t*>(arena_ + vs_off_));
    launches_ += 3;
    TCG_CUDA(cudaGetLastError());
    if (prof_) { prof_->ema.emplace_back(b0, prof_->used); TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
  }
  struct Marks { size_t t0, t1, t2; };
  std::vector<Marks> marks;
  for (auto& e : exec_) {
    Marks m{0, 0, 0};
    if (stats) m.t0 = mark();
    if (e.dup_of >= 0) {  // identical to an earlier node: its table is aliased
      if (stats) { m.t1 = mark(); m.t2 = mark(); }
      marks.push_back(m);
      continue;
    }
    const float* P = H;
    if (e.pp_dup_of >= 0) {
      P = table_ptr(e.pp_off);
    } else if (!e.p_leaf && n_ > 0) {
      size_t p0 = 0;
      if (prof_) { p0 = prof_->used; TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
      if (e.rooted && e.pstream) {
        rooted_spmm(e, table_ptr(table_off_[e.p]), table_ptr(e.pp_off), d_colors, table_ptr(e.out_off));
      } else if (e.rooted) {
        rooted_spmm(e, table_ptr(table_off_[e.p]), table_ptr(e.pp_off), d_colors);
      } else {
        spmm(table_ptr(table_off_[e.p]), table_ptr(e.pp_off), e.Cp);
      }
      if (prof_) { prof_->spmm.emplace_back(p0, prof_->used); TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
      P = table_ptr(e.pp_off);
    }
    if (e.virt) {
      if (stats) { m.t1 = mark(); m.t2 = mark(); }
      marks.push_back(m);
      continue;
    }
    if (stats) m.t1 = mark();
    size_t q0 = 0;
    if (prof_) { q0 = prof_->used; TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
    const float* A = e.a_leaf ? nullptr : table_ptr(table_off_[e.a]);
    if (n_ > 0 && rooted_ema_ && e.pstream) {
      // (the SpMM wrote the output)
    } else if (n_ > 0 && rooted_ema_) {
      launch_rt_ema(e, A, P, d_root_acc);
      ++launches_;
      TCG_CUDA(cudaGetLastError());
    } else if (n_ > 0) {
      const unsigned vgrid = static_cast<unsigned>(std::min<int64_t>(n_, 148 * 16));
      if (e.vtx) {
        auto smem_attr = [&](const void* f) {
          smem_limit(f, e.vtx_smem);
        };
        if (e.root) {
          double* rout = reinterpret_cast<double*>(arena_ + e.out_off);
          smem_attr(reinterpret_cast<const void*>(dev::ema_vtx_root));
          dev::ema_vtx_root<<<vgrid, 256, e.vtx_smem, stream_>>>(A, P, d_colors, e.d_split, e.pairs, e.Ca, e.Cps,
                                                                   e.a_leaf ? 1 : 0, n_, rout, d_root_acc);
        } else if (e.a_leaf) {
          smem_attr(reinterpret_cast<const void*>(dev::ema_vtx_aleaf));
          dev::ema_vtx_aleaf<<<vgrid, 256, e.vtx_smem, stream_>>>(P, d_colors, e.d_drop, plan_.k, e.Cps, e.Cs, n_,
                                                                    table_ptr(e.out_off));
        } else {
          smem_attr(reinterpret_cast<const void*>(dev::ema_vtx_blocked));
          dev::ema_vtx_blocked<<<vgrid, 256, e.vtx_smem, stream_>>>(
              A, P, static_cast<const dev::GroupDesc*>(e.d_groups), e.ngroups,
              static_cast<const dev::BlockDesc*>(e.d_blocks), e.Ca, e.Cp, e.Cs, n_, table_ptr(e.out_off),
              e.Cps, e.rooted ? e.d_pinv : nullptr);
        }
      } else if (e.root) {
        double* rout = reinterpret_cast<double*>(arena_ + e.out_off);
        if (e.a_leaf) {
          if (e.ema_staged) launch_root<true, true>(e, stream_, n_, A, P, d_colors, rout, d_root_acc, d_tile_tot_);
          else launch_root<true, false>(e, stream_, n_, A, P, d_colors, rout, d_root_acc, d_tile_tot_);
        } else {
          if (e.ema_staged) launch_root<false, true>(e, stream_, n_, A, P, d_colors, rout, d_root_acc, d_tile_tot_);
          else launch_root<false, false>(e, stream_, n_, A, P, d_colors, rout, d_root_acc, d_tile_tot_);
        }
      } else {
        float* out = table_ptr(e.out_off);
        if (e.a_leaf) {
          if (e.ema_staged) launch_node<true, true>(e, plan_.k, stream_, n_, A, P, d_colors, out);
          else launch_node<true, false>(e, plan_.k, stream_, n_, A, P, d_colors, out);
        } else if (e.blocked) {
          auto kern = dev::ema_blocked<true>;
          smem_limit(reinterpret_cast<const void*>(kern), e.ema_smem);
          kern<<<static_cast<unsigned>((n_ + dev::kTileV - 1) / dev::kTileV), 256, e.ema_smem, stream_>>>(
              A, P, static_cast<const dev::GroupDesc*>(e.d_groups), e.ngroups,
              static_cast<const dev::BlockDesc*>(e.d_blocks), e.Ca, e.Cp, e.Cs, n_, out, e.Cps,
              e.rooted ? e.d_pinv : nullptr);
        } else {
          if (e.ema_staged) launch_node<false, true>(e, plan_.k, stream_, n_, A, P, d_colors, out);
          else launch_node<false, false>(e, plan_.k, stream_, n_, A, P, d_colors, out);
        }
      }
      ++launches_;
      TCG_CUDA(cudaGetLastError());
    }
    if (prof_) { prof_->ema.emplace_back(q0, prof_->used); TCG_CUDA(cudaEventRecord(prof_->get(), stream_)); }
    if (stats) m.t2 = mark();
    marks.push_back(m);
  }
  if (n_ > 0 && !exec_.empty() && d_total) {
    // fixed-shape fp64 sum of the per-vertex root counts (internal row order;
    // one segment per copy when this is a batch engine)
    ensure_tile_tot(static_cast<int64_t>(batch_copies_) * dev::kRootChunks);
    dev::root_partial<<<batch_copies_ * dev::kRootChunks, 256, 0, stream_>>>(
        reinterpret_cast<const double*>(arena_ + exec_.back().out_off), n_ / batch_copies_, d_tile_tot_);
    dev::root_reduce<<<batch_copies_, 64, 0, stream_>>>(d_tile_tot_, dev::kRootChunks, d_total);
    launches_ += 2;
  } else if (d_total) {
    TCG_CUDA(cudaMemsetAsync(d_total, 0, sizeof(double), stream_));
  }
  TCG_CUDA(cudaGetLastError());
  if (stats) {
    TCG_CUDA(cudaStreamSynchronize(stream_));
    const Binom& B = binom();
    for (int i = 0; i < plan_.num_nodes; ++i) stats[i] = tcg_node_stats{};
    for (size_t i = 0; i < exec_.size(); ++i) {
      const NodeExec& e = exec_[i];
      float s1 = 0, s2 = 0;
      TCG_CUDA(cudaEventElapsedTime(&s1, ev[marks[i].t0], ev[marks[i].t1]));
      TCG_CUDA(cudaEventElapsedTime(&s2, ev[marks[i].t1], ev[marks[i].t2]));
      tcg_node_stats& st = stats[e.id];
      st.spmm_seconds = s1 * 1e-3;
      st.ema_seconds = s2 * 1e-3;
      st.seconds = st.spmm_seconds + st.ema_seconds;
      st.neighbor_passes = static_cast<uint64_t>(e.Cp);
      st.traversals = static_cast<uint64_t>(e.Cp) * static_cast<uint64_t>(n_);
      const uint64_t pairs_total = static_cast<uint64_t>(e.Cs) * static_cast<uint64_t>(B(e.size, e.sa));
      st.flops = static_cast<uint64_t>(e.Cp) * static_cast<uint64_t>(nnz_) + 2ull * n_ * pairs_total;
      st.spmm_bytes = 4ull * nnz_ + 8ull * (n_ + 1) + 8ull * n_ * static_cast<uint64_t>(e.Cp);
      st.ema_bytes = 4ull * n_ * ((e.a_leaf ? 0ull : static_cast<uint64_t>(e.Ca)) + e.Cp) +
                     (e.root ? 8ull * n_ : 4ull * n_ * static_cast<uint64_t>(e.Cs));
      st.ema_flops = 2ull * n_ * pairs_total;
    }
  }
  for (auto e : ev) cudaEventDestroy(e);
}

double Engine::run_coloring(uint64_t seed, const uint8_t* host_colors, double* per_vertex,
                            tcg_node_stats* stats) {
  TCG_CUDA(cudaSetDevice(cfg_.device));
  ensure_arena();
  ensure_colors(nglob_);
  if (host_colors) {
    for (int32_t i = 0; i < nglob_; ++i)
      if (host_colors[i] >= plan_.k) throw invalid_argument("coloring value out of range [0, k)");
    TCG_CUDA(cudaMemcpyAsync(d_colors_, host_colors, nglob_, cudaMemcpyHostToDevice, stream_));
  }
  const uint8_t* dc = host_colors ? d_colors_ : take_or_generate(seed);
  if (!host_colors) prefetch_next(seed + 1);  // (overlaps this coloring's DP)
  run_dp(dc, d_scalars_, nullptr, stats);
  double total = 0;
  TCG_CUDA(cudaMemcpyAsync(&total, d_scalars_, sizeof(double), cudaMemcpyDeviceToHost, stream_));
  if (per_vertex && nglob_ > 0) {
    if (exec_.empty()) {
      for (int32_t i = 0; i < nglob_; ++i) per_vertex[i] = 1.0;  // k = 1: every vertex once
    } else if (sharded()) {
      gather_per_vertex(reinterpret_cast<const double*>(arena_ + exec_.back().out_off), per_vertex);
    } else {
      unpermute_to_host(reinterpret_cast<const double*>(arena_ + exec_.back().out_off), per_vertex);
    }
  }
  if (cfg_.flags & TCG_KEEP_TABLES) {
    last_colors_.resize(nglob_);
    TCG_CUDA(cudaMemcpyAsync(last_colors_.data(), dc, nglob_, cudaMemcpyDeviceToHost, stream_));
  }
  TCG_CUDA(cudaStreamSynchronize(stream_));
  if (exec_.empty()) total = static_cast<double>(nloc_);
  finish_shard_totals(&total, 1);
  tables_valid_ = true;
  if (!std::isfinite(total)) throw nonfinite_error("rooted total is not finite (fp64 overflow)");
  return total;
}

static int color_chunk(int count, int32_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(
      {static_cast<int64_t>(count), 1024, std::max<int64_t>(1, (int64_t{1} << 30) / std::max(n, 1))})));
}

void Engine::estimate(uint64_t seed, int iterations, double* totals, double* est, double* se,
                      double* per_vertex_est) {
  if (iterations < 1) throw invalid_argument("iterations must be >= 1");
  static const bool timing = std::getenv("TCG_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto since = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
  TCG_CUDA(cudaSetDevice(cfg_.device));
  ensure_arena();
  const int chunk = color_chunk(iterations, nglob_);
  ensure_colors(static_cast<int64_t>(chunk) * nglob_);
  if (est_tot_cap_ < iterations) {
    dfree(d_est_tot_);
    est_tot_cap_ = 0;
    TCG_CUDA(cudaMalloc(&d_est_tot_, sizeof(double) * iterations));
    est_tot_cap_ = iterations;
  }
  double* d_totals = d_est_tot_;
  double* d_acc = nullptr;
  {
    if (per_vertex_est && !exec_.empty()) {
      if (est_acc_cap_ < std::max(n_, 1)) {
        dfree(d_est_acc_);
        est_acc_cap_ = 0;
        TCG_CUDA(cudaMalloc(&d_est_acc_, sizeof(double) * std::max(n_, 1)));
        est_acc_cap_ = std::max(n_, 1);
      }
      d_acc = d_est_acc_;
      TCG_CUDA(cudaMemsetAsync(d_acc, 0, sizeof(double) * std::max(n_, 1), stream_));
    }
    std::vector<uint64_t> seeds(chunk);
    for (int i0 = 0; i0 < iterations; i0 += chunk) {
      const int c = std::min(chunk, iterations - i0);
      for (int j = 0; j < c; ++j) seeds[j] = seed + static_cast<uint64_t>(i0 + j);
      gen_colors(seeds.data(), c, d_colors_);
      for (int j = 0; j < c;) {
        const int B = pick_batch(c - j);
        if (B > 1) run_batch(d_colors_ + static_cast<int64_t>(j) * nglob_, B, d_totals + i0 + j, d_acc);
        else run_dp(d_colors_ + static_cast<int64_t>(j) * nglob_, d_totals + i0 + j, d_acc, nullptr);
        j += B;
      }
    }
    if (timing) {
      const double q = since();
      TCG_CUDA(cudaStreamSynchronize(stream_));
      std::fprintf(stderr, "[tcg timing] estimate: enqueue %.1f ms, device done %.1f ms\n", q, since());
    }
    TCG_CUDA(cudaMemcpyAsync(totals, d_totals, sizeof(double) * iterations, cudaMemcpyDeviceToHost, stream_));
    std::vector<double> acc;
    if (d_acc) {
      acc.resize(nglob_);
      if (sharded()) {
        gather_per_vertex(d_acc, acc.data());
      } else {
        unpermute_to_host(d_acc, acc.data());
      }
    }
    TCG_CUDA(cudaStreamSynchronize(stream_));
    if (exec_.empty())
      for (int i = 0; i < iterations; ++i) totals[i] = static_cast<double>(nloc_);
    finish_shard_totals(totals, iterations);
    // estimator.hpp:80-91, same arithmetic order
    double mean = 0.0;
    for (int i = 0; i < iterations; ++i) mean += totals[i];
    mean /= static_cast<double>(iterations);
    double var = 0.0;
    for (int i = 0; i < iterations; ++i) var += (totals[i] - mean) * (totals[i] - mean);
    const double scale = 1.0 / (static_cast<double>(aut_) * colorful_probability(plan_.k));
    *est = mean * scale;
    *se = iterations > 1 ? std::sqrt(var / (static_cast<double>(iterations) *
                                            static_cast<double>(iterations - 1))) * scale
                         : 0.0;
    if (per_vertex_est) {
      for (int32_t v = 0; v < nglob_; ++v)
        per_vertex_est[v] = (exec_.empty() ? 1.0 : acc[v] / iterations) * scale;
    }
    for (int i = 0; i < iterations; ++i)
      if (!std::isfinite(totals[i])) throw nonfinite_error("rooted total is not finite (fp64 overflow)");
  }
  if (timing) std::fprintf(stderr, "[tcg timing] estimate: total %.1f ms\n", since());
  tables_valid_ = false;
}

// ------------------------------------------------------- batched colorings
// Batch size for `count` pending colorings: small graphs only (the union of
// B copies <= 2^20 rows and 2^26 entries, its tables <= 8 GB), B <= 64.
int Engine::pick_batch(int count) const {
  static const int mode = [] {
    const char* s = std::getenv("TCG_BATCH");
    return s ? std::atoi(s) : 1;
  }();
  if (!mode || count < 2 || sharded() || n_ <= 0 || exec_.empty() || batch_copies_ > 1) return 1;
  // part schedules depend on the gather source's size (colour-class parts,
  // vertex-range parts of the full-table SpMM): a union would cut, and round,
  // differently -- keep those plans unbatched so results stay bit-identical
  if (rooted_parts_ > 1) return 1;
  for (const auto& e : exec_)
    if (!e.p_leaf && !e.rooted && e.dup_of < 0 && e.pp_dup_of < 0) return 1;
  int64_t B = std::min<int64_t>({count, 64, (int64_t{1} << 20) / n_, (int64_t{1} << 26) / std::max<int64_t>(nnz_, 1),
                                 (int64_t{8} << 30) / std::max<int64_t>(arena_bytes_ + partial_bytes_, 1)});
  if (cfg_.memory_budget > 0)  // the union's tables count against the caller's budget too
    B = std::min<int64_t>(B, cfg_.memory_budget / std::max<int64_t>(arena_bytes_, 1));
  return B >= 2 ? static_cast<int>(B) : 1;
}

// The engine over the B-fold union of this engine's (internal) graph, same
// template, same stream; rebuilt when the graph, the template or B changes.
Engine* Engine::batch_engine(int B) {
  // one engine per batch size in use (a handful at most: estimate/time calls
  // with different counts do not rebuild each other's union)
  Batch* slot = nullptr;
  for (auto& x : batches_)
    if (x.B == B) slot = &x;
  if (slot && slot->tpl_gen != tpl_gen_) {
    slot->eng.reset();
    slot->graph_gen = ~0ull;
  }
  if (!slot) {
    if (batches_.size() >= 4) batches_.erase(batches_.begin());  // oldest
    batches_.push_back(Batch{B, nullptr, ~0ull, ~0ull});
    slot = &batches_.back();
  }
  if (!slot->eng) {
    tcg_config c = cfg_;
    c.flags &= ~TCG_KEEP_TABLES;
    c.memory_budget = 0;
    auto be = std::make_unique<Engine>(c, stream_);
    be->no_relabel_ = true;
    be->batch_copies_ = B;
    be->limit_override_ = limit_override_;
    std::vector<int32_t> edges;
    for (const auto& pr : tpl_.edges) {
      edges.push_back(pr.first);
      edges.push_back(pr.second);
    }
    be->set_template(tpl_.k, edges.data(), tpl_.root);
    slot->eng = std::move(be);
    slot->tpl_gen = tpl_gen_;
    slot->graph_gen = ~0ull;
  }
  if (slot->graph_gen != graph_gen_) {
    // the union of this graph's copies, built on the device in scratch kept
    // across graphs (e2e: a new CSR per call), then handed to the batch engine
    const int64_t nU = static_cast<int64_t>(n_) * B, eU = nnz_ * B;
    if (urp_cap_ < nU + 1) {
      dfree(d_urp_);
      urp_cap_ = 0;
      TCG_CUDA(cudaMalloc(&d_urp_, sizeof(int64_t) * (nU + 1)));
      urp_cap_ = nU + 1;
    }
    if (ucol_cap_ < std::max<int64_t>(eU, 1)) {
      dfree(d_ucol_);
      ucol_cap_ = 0;
      TCG_CUDA(cudaMalloc(&d_ucol_, sizeof(int32_t) * std::max<int64_t>(eU, 1)));
      ucol_cap_ = std::max<int64_t>(eU, 1);
    }
    dev::union_graph<<<148 * 4, 256, 0, stream_>>>(d_row_ptr_, d_col_, n_, nnz_, B, d_urp_, d_ucol_);
    TCG_CUDA(cudaGetLastError());
    slot->eng->set_graph_ptrs(static_cast<int32_t>(nU), d_urp_, d_ucol_, false, eU);
    slot->eng->ensure_arena();
    slot->graph_gen = graph_gen_;
  }
  return slot->eng.get();
}

// B colorings (caller order) as one DP over the union: the copies' totals
// (fixed-shape per-copy reductions == run_dp's) and per-vertex accumulation
// in coloring order, so results equal B separate run_dp calls bit for bit.
void Engine::run_batch(const uint8_t* d_colors, int B, double* d_totals, double* d_acc) {
  Engine* be = batch_engine(B);
  be->ensure_colors(static_cast<int64_t>(n_) * B);
  dev::batch_colors<<<static_cast<unsigned>((static_cast<int64_t>(n_) * B + 255) / 256), 256, 0, stream_>>>(
      d_colors, nglob_, relabeled_ ? d_perm_ : nullptr, n_, B, be->d_colors_);
  ++launches_;
  be->prof_ = prof_;
  const int64_t l0 = be->launches_;
  be->run_dp(be->d_colors_, d_totals, nullptr, nullptr);
  be->prof_ = nullptr;
  launches_ += be->launches_ - l0;
  if (d_acc) {
    dev::fold_copies<<<static_cast<unsigned>((n_ + 255) / 256), 256, 0, stream_>>>(
        reinterpret_cast<const double*>(be->arena_ + be->exec_.back().out_off), n_, B, d_acc);
    ++launches_;
  }
  TCG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------ bench timing
cudaEvent_t Engine::Prof::get() {
  if (used == pool.size()) {
    cudaEvent_t e;
    TCG_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}

void Engine::time_colorings(uint64_t seed, int count, bool per_kernel, double* totals,
                            tcg_timing* out) {
  if (count < 1) throw invalid_argument("count must be >= 1");
  TCG_CUDA(cudaSetDevice(cfg_.device));
  ensure_arena();
  const int chunk = color_chunk(count, nglob_);
  ensure_colors(static_cast<int64_t>(chunk) * nglob_);
  double* d_totals = nullptr;
  TCG_CUDA(cudaMalloc(&d_totals, sizeof(double) * count));
  Prof prof;
  cudaEvent_t e0, e1;
  TCG_CUDA(cudaEventCreate(&e0));
  TCG_CUDA(cudaEventCreate(&e1));
  const int64_t l0 = launches_;
  std::vector<uint64_t> seeds(chunk);
  try {
    if (per_kernel) prof_ = &prof;
    TCG_CUDA(cudaStreamSynchronize(stream_));
    TCG_CUDA(cudaEventRecord(e0, stream_));
    for (int i0 = 0; i0 < count; i0 += chunk) {
      const int c = std::min(chunk, count - i0);
      for (int j = 0; j < c; ++j) seeds[j] = seed + static_cast<uint64_t>(i0 + j);
      gen_colors(seeds.data(), c, d_colors_);
      for (int j = 0; j < c;) {
        const int B = pick_batch(c - j);
        if (B > 1) run_batch(d_colors_ + static_cast<int64_t>(j) * nglob_, B, d_totals + i0 + j, nullptr);
        else run_dp(d_colors_ + static_cast<int64_t>(j) * nglob_, d_totals + i0 + j, nullptr, nullptr);
        j += B;
      }
    }
    TCG_CUDA(cudaEventRecord(e1, stream_));
    TCG_CUDA(cudaEventSynchronize(e1));
    prof_ = nullptr;
  } catch (...) {
    prof_ = nullptr;
    dfree(d_totals);
    throw;
  }
  tcg_timing t{};
  float ms = 0;
  TCG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  t.total_ms = ms;
  for (auto& pr : prof.spmm) {
    TCG_CUDA(cudaEventElapsedTime(&ms, prof.pool[pr.first], prof.pool[pr.second]));
    t.spmm_ms += ms;
  }
  for (auto& pr : prof.ema) {
    TCG_CUDA(cudaEventElapsedTime(&ms, prof.pool[pr.first], prof.pool[pr.second]));
    t.ema_ms += ms;
  }
  for (auto ev : prof.pool) cudaEventDestroy(ev);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  t.launches = launches_ - l0;
  const Binom& B = binom();
  const double n = n_, nnz = static_cast<double>(nnz_);
  for (auto& e : exec_) {
    if (e.dup_of >= 0) continue;  // not executed (aliased): no work claimed
    if (!e.p_leaf && e.pp_dup_of < 0) {
      t.spmm_launches += count;
      t.spmm_alg_bytes += count * (4 * nnz + 8 * (n + 1) + 8 * n * e.Cp);
      // columns actually gathered per neighbour; the rooted SpMMs never walk
      // a row's own-color neighbours (expected 1/k of them)
      const int32_t gc = e.rooted ? e.rl_groups * e.rl_zw : e.Cp;
      const double walked = e.rooted ? nnz * (plan_.k - 1) / plan_.k : nnz;
      t.spmm_gathered_bytes += count * walked * 4.0 * (static_cast<double>(dev::num_panels(gc) - 1) * dev::kZ +
                                                        dev::last_panel_width(gc));
    }
    if (e.virt) continue;  // no eMA executed: no eMA work claimed
    t.ema_launches += count;
    t.ema_alg_bytes += count * (4 * n * ((e.a_leaf ? 0 : e.Ca) + e.Cp) + (e.root ? 8 * n : 4 * n * e.Cs));
    t.ema_flops += count * 2 * n * e.Cs * static_cast<double>(B(e.size, e.sa));
  }
  if (need_hist_) t.hist_alg_bytes = count * (4 * nnz + 8 * (n + 1) + n + 4 * n * plan_.k);
  std::vector<double> h(count);
  copy_sync(h.data(), d_totals, sizeof(double) * count, cudaMemcpyDeviceToHost);
  dfree(d_totals);
  if (exec_.empty()) std::fill(h.begin(), h.end(), static_cast<double>(nloc_));
  finish_shard_totals(h.data(), count);
  if (totals) std::copy(h.begin(), h.end(), totals);
  for (double x : h)
    if (!std::isfinite(x)) throw nonfinite_error("rooted total is not finite (fp64 overflow)");
  *out = t;
  tables_valid_ = false;
}

// ------------------------------------------------------------ inspection
static void unpanel(const std::vector<float>& t, int64_t n, int64_t C, double* out) {
  for (int64_t v = 0; v < n; ++v)
    for (int64_t c = 0; c < C; ++c) out[v * C + c] = t[dev::panel_offset(C, n, v, c)];
}

void Engine::node_table(int id, int which, double* out) {
  if (sharded()) throw invalid_argument("node tables are not inspectable on a sharded context");
  if (!(cfg_.flags & TCG_KEEP_TABLES)) throw invalid_argument("context not created with TCG_KEEP_TABLES");
  if (!tables_valid_) throw invalid_argument("no coloring has been run since the last change");
  if (id < 0 || id >= plan_.num_nodes) throw invalid_argument("node id out of range");
  const int64_t k = plan_.k;
  if (plan_.is_leaf(id) && which == 0) {  // the one-hot leaf table, caller order
    std::fill(out, out + static_cast<int64_t>(nglob_) * k, 0.0);
    for (int64_t v = 0; v < nglob_; ++v) out[v * k + last_colors_[v]] = 1.0;
    return;
  }
  if (!relabeled_) {
    node_table_internal(id, which, out, last_colors_);
    return;
  }
  // internal rows -> the caller's vertices (isolated vertices: zero rows)
  const int64_t C = plan_.is_leaf(id) ? k : id == plan_.full_node() ? 1 : binom()(plan_.k, plan_.size[id]);
  const std::vector<int32_t> perm = host_perm();
  std::vector<uint8_t> lc(static_cast<size_t>(n_));
  for (int32_t i = 0; i < n_; ++i) lc[i] = last_colors_[perm[i]];
  std::vector<double> tmp(static_cast<size_t>(n_) * C);
  node_table_internal(id, which, tmp.data(), lc);
  std::fill(out, out + static_cast<int64_t>(nglob_) * C, 0.0);
  for (int32_t i = 0; i < n_; ++i) std::copy(tmp.begin() + i * C, tmp.begin() + (i + 1) * C, out + perm[i] * C);
}

void Engine::node_table_internal(int id, int which, double* out, const std::vector<uint8_t>& lc) {
  const int64_t n = n_, k = plan_.k;
  if (plan_.is_leaf(id)) {
    if (hist_off_ < 0) throw invalid_argument("no neighbour histogram in this plan");
    std::vector<float> h(dev::table_floats(k, n));
    copy_sync(h.data(), arena_ + hist_off_, h.size() * 4, cudaMemcpyDeviceToHost);
    unpanel(h, n, k, out);
    return;
  }
  const int64_t C = binom()(plan_.k, plan_.size[id]);
  if (id == plan_.full_node()) {
    if (which != 0) throw invalid_argument("the root has no SpMM output");
    copy_sync(out, arena_ + table_off_[id], sizeof(double) * n, cudaMemcpyDeviceToHost);
    return;
  }
  const int64_t off = which == 0 ? table_off_[id] : pprime_off_[id];
  if (off < 0) throw invalid_argument("table not available for this node");
  if (which == 0 && rooted_ema_) {
    // rooted table (RR or the SpMM slot layout): expand to the full C(k,s)
    // columns, zero wherever the set misses the vertex's color
    for (const auto& e : exec_) {
      if (e.id != id) continue;
      const int s = plan_.size[id];
      std::vector<float> t(dev::table_floats(e.Cout, n));
      copy_sync(t.data(), arena_ + off, t.size() * 4, cudaMemcpyDeviceToHost);
      std::vector<int64_t> rel(static_cast<size_t>(C) * k, -1);  // [S][c] relabeled index or -1
      int cs[kMaxK];
      for (int64_t S = 0; S < C; ++S) {
        set_of(plan_.k, S, s, cs);
        for (int j = 0; j < s; ++j) rel[static_cast<size_t>(S) * k + cs[j]] = relabeled_index(cs, s, cs[j]);
      }
      std::vector<int32_t> qof(e.amap_host.size());
      for (int c = 0; c < k && !e.amap_host.empty(); ++c)
        for (int32_t q = 0; q < e.Ws; ++q) qof[static_cast<size_t>(c) * e.Ws + e.amap_host[static_cast<size_t>(c) * e.Ws + q]] = q;
      for (int64_t v = 0; v < n; ++v) {
        const int c = lc[v];
        for (int64_t S = 0; S < C; ++S) {
          const int64_t j = rel[static_cast<size_t>(S) * k + c];
          double x = 0.0;
          if (j >= 0 && e.pstream && e.omap.empty())  // packed: q with amap[c][q] == j
            x = t[dev::panel_offset(e.Cout, n, v, qof[static_cast<size_t>(c) * e.Ws + j])];
          else if (j >= 0)
            x = e.omap.empty() ? t[dev::panel_offset(e.Cout, n, v, j)]
                               : t[dev::panel_offset(e.Cout, n, v, e.omap[static_cast<size_t>(c) * e.Ws + j])];
          out[v * C + S] = x;
        }
      }
      return;
    }
  }
  if (which == 1) {
    for (const auto& e : exec_)
      if (e.p == id && e.rooted) {  // group-major P': storage column perm[S]
        std::vector<float> t(dev::table_floats(e.Cps, n));
        copy_sync(t.data(), arena_ + off, t.size() * 4, cudaMemcpyDeviceToHost);
        // columns containing c(v) are not computed by the rooted SpMM (never
        // consumed): exported as 0
        const int sp = plan_.size[id];
        std::vector<uint32_t> mask(static_cast<size_t>(C));
        int cs[kMaxK];
        for (int64_t c = 0; c < C; ++c) {
          set_of(plan_.k, c, sp, cs);
          uint32_t m = 0;
          for (int j = 0; j < sp; ++j) m |= 1u << cs[j];
          mask[static_cast<size_t>(c)] = m;
        }
        std::vector<int64_t> rel;  // pair layout: [S][c] relabeled index of S past c
        if (e.pair) {
          rel.assign(static_cast<size_t>(C) * k, -1);
          for (int64_t c = 0; c < C; ++c) {
            set_of(plan_.k, c, sp, cs);
            for (int q = 0; q < k; ++q)
              if (!(mask[static_cast<size_t>(c)] >> q & 1u)) {
                int tt[kMaxK];
                for (int j = 0; j < sp; ++j) tt[j] = cs[j] > q ? cs[j] - 1 : cs[j];
                rel[static_cast<size_t>(c) * k + q] = index_of(tt, sp);
              }
          }
        }
        for (int64_t v = 0; v < n; ++v)
          for (int64_t c = 0; c < C; ++c) {
            const int cv = lc[v];
            if (mask[static_cast<size_t>(c)] >> cv & 1u) { out[v * C + c] = 0.0; continue; }
            const int64_t col = e.pair ? e.rl_perm[rel[static_cast<size_t>(c) * k + cv]] : e.rl_perm[c];
            out[v * C + c] = t[dev::panel_offset(e.Cps, n, v, col)];
          }
        return;
      }
  }
  std::vector<float> t(dev::table_floats(C, n));
  copy_sync(t.data(), arena_ + off, t.size() * 4, cudaMemcpyDeviceToHost);
  unpanel(t, n, C, out);
}

void Engine::spmm_host(const float* x, int cols, float* y) {
  if (n_ < 0) throw invalid_argument("no graph set (tcg_set_graph)");
  if (sharded()) throw invalid_argument("tcg_spmm is not available on a sharded context");
  if (cols < 1) throw invalid_argument("cols must be >= 1");
  TCG_CUDA(cudaSetDevice(cfg_.device));
  const int64_t n = n_;
  for (int p = 0; p < dev::num_panels(cols); ++p) ensure_schedules(parts_for_width(dev::panel_width(cols, p)));
  const std::vector<int32_t> perm = host_perm();  // internal row -> caller vertex
  std::vector<float> xp(dev::table_floats(cols, n), 0.f);
  for (int64_t v = 0; v < n; ++v)
    for (int64_t c = 0; c < cols; ++c) xp[dev::panel_offset(cols, n, v, c)] = x[perm[v] * cols + c];
  float *dx = nullptr, *dy = nullptr;
  double* saved_partial = d_partial_;
  double* dp = nullptr;
  try {
    TCG_CUDA(cudaMalloc(&dx, std::max<size_t>(xp.size() * 4, 4)));
    TCG_CUDA(cudaMalloc(&dy, std::max<size_t>(xp.size() * 4, 4)));
    if (max_slots_) TCG_CUDA(cudaMalloc(&dp, static_cast<size_t>(max_slots_) * dev::kZ * 8));
    copy_sync(dx, xp.data(), xp.size() * 4, cudaMemcpyHostToDevice);
    d_partial_ = dp;
    if (n > 0) spmm(dx, dy, cols);
    d_partial_ = saved_partial;
    TCG_CUDA(cudaStreamSynchronize(stream_));
    copy_sync(xp.data(), dy, xp.size() * 4, cudaMemcpyDeviceToHost);
  } catch (...) {
    d_partial_ = saved_partial;
    dfree(dx); dfree(dy); dfree(dp);
    throw;
  }
  dfree(dx); dfree(dy); dfree(dp);
  std::fill(y, y + static_cast<int64_t>(nglob_) * cols, 0.f);  // isolated vertices: 0
  for (int64_t v = 0; v < n; ++v)
    for (int64_t c = 0; c < cols; ++c) y[perm[v] * cols + c] = xp[dev::panel_offset(cols, n, v, c)];
}

// Kernel-level hook of the PRODUCTION rooted SpMM (tcg_spmm_rooted): one
// passive table M (n x C(k, s), caller order, rooted: M[u, S] = 0 unless
// c(u) is in S) through exactly the per-coloring path a DP node runs --
// bucket_coloring (rotated colour order, hub-row chunks), the k-colour slot
// layout (spmm_rooted<zw, 4, false>) or the pair layout (pair_expand +
// spmm_rooted<zw, 4, true>), rooted_fixup for rows split into segments --
// and Y[v, T] = sum over u in N(v) of M[u, T] for every T missing c(v) (the
// columns any eMA consumes; 0 elsewhere).  la_kernels.hpp:83-102 semantics.
void Engine::spmm_rooted_host(int k, int s, bool pair, const uint8_t* colors, const float* x, float* y) {
  if (n_ < 0) throw invalid_argument("no graph set (tcg_set_graph)");
  if (sharded()) throw invalid_argument("tcg_spmm_rooted is not available on a sharded context");
  if (k < 2 || k > kMaxK || s < 1 || s >= k) throw invalid_argument("need 2 <= k <= 20 and 1 <= s < k");
  if (pair && k < 3) throw invalid_argument("the pair layout needs k >= 3");
  TCG_CUDA(cudaSetDevice(cfg_.device));
  const Binom& B = binom();
  const int64_t n = n_, C = B(k, s);
  for (int32_t v = 0; v < nglob_; ++v)
    if (colors[v] >= k) throw invalid_argument("coloring value out of range [0, k)");
  const std::vector<int32_t> perm = host_perm();
  std::vector<uint8_t> lc(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) lc[i] = colors[perm[i]];
  int cs[kMaxK];
  NodeExec e;
  e.id = -1;
  e.p = -1;
  e.sp = s;
  e.rooted = true;
  e.pair = pair;
  const RootedLayout rl = build_rooted_layout(pair ? k - 1 : k, s);
  e.Cps = rl.store_cols;
  e.rl_zw = rl.zw;
  e.rl_groups = rl.groups;
  e.rl_fbase = rl.fbase;
  e.rl_fsize = rl.fsize;
  e.rl_perm = rl.perm;
  e.slot_K = pair ? k - 1 : k;
  int fpad_max = 0;
  for (int g = 0; g < rl.groups; ++g)
    fpad_max = std::max(fpad_max, (g + 1 < rl.groups ? rl.fbase[g + 1] : rl.store_cols) - rl.fbase[g]);
  e.rooted_smem = static_cast<size_t>(dev::kSpmmWarps) * (128 / rl.zw) * (fpad_max + 4) * 4 + 2 * (e.slot_K + 1) * rl.zw;
  const int slots = rl.groups * rl.zw;
  // input: the k-colour slot layout (groups x zw columns), or RR (pair)
  const int64_t wx = B(k - 1, s - 1);
  const int64_t in_cols = pair ? wx : slots;
  std::vector<float> xin(dev::table_floats(in_cols, n), 0.f);
  std::vector<int16_t> xm;
  if (pair) {
    e.Wx = static_cast<int32_t>(wx);
    xm.assign(static_cast<size_t>(k) * k * slots, -1);
    for (int cu = 0; cu < k; ++cu)
      for (int cv = 0; cv < k; ++cv) {
        if (cu == cv) continue;
        const int cr = cu - (cu > cv ? 1 : 0);
        for (int i = 0; i < slots; ++i) {
          const int32_t col1 = rl.slot_col[static_cast<size_t>(cr) * slots + i];
          if (col1 < 0) continue;
          set_of(k - 1, col1, s, cs);
          for (int q = 0; q < s; ++q) cs[q] = cs[q] >= cv ? cs[q] + 1 : cs[q];
          xm[(static_cast<size_t>(cu) * k + cv) * slots + i] = static_cast<int16_t>(relabeled_index(cs, s, cu));
        }
      }
    for (int64_t u = 0; u < n; ++u) {  // RR column j of u = M[u, (set j past c(u)) + c(u)]
      const int cu = lc[u];
      for (int64_t j = 0; j < wx; ++j) {
        set_of(k - 1, j, s - 1, cs);
        int t[kMaxK], m = 0;
        bool put = false;
        for (int q = 0; q < s - 1; ++q) {
          const int c = cs[q] >= cu ? cs[q] + 1 : cs[q];
          if (!put && c > cu) { t[m++] = cu; put = true; }
          t[m++] = c;
        }
        if (!put) t[m++] = cu;
        xin[dev::panel_offset(in_cols, n, u, j)] = x[static_cast<int64_t>(perm[u]) * C + index_of(t, s)];
      }
    }
  } else {
    for (int64_t u = 0; u < n; ++u)
      for (int i = 0; i < slots; ++i) {
        const int32_t col = rl.slot_col[static_cast<size_t>(lc[u]) * slots + i];
        if (col >= 0) xin[dev::panel_offset(in_cols, n, u, i)] = x[static_cast<int64_t>(perm[u]) * C + col];
      }
  }
  // scratch arena for this call (the engine's own arena and offsets are restored)
  const int psave = rooted_parts_;
  char* asave = arena_;
  const int64_t o_rc = rcol_off_, o_cut = rcut_off_, o_lc = lcnt_off_, o_seg = pseg_off_, o_key = pkey_off_,
                o_perm = pperm_off_, o_cnt = pcnt_off_;
  double* part_save = d_partial_;
  const int64_t nseg = sched_.at(1)[0].nseg_padded;
  ArenaPlanner ap;
  rcol_off_ = ap.alloc(4 * std::max<int64_t>(nnz_, 1));
  rcut_off_ = ap.alloc(8 * n * 2);
  lcnt_off_ = ap.alloc(4 * 32 * static_cast<int64_t>(std::max(nlchunks_, 1)));
  pseg_off_ = ap.alloc(static_cast<int64_t>(sizeof(dev::Seg)) * nseg);
  pkey_off_ = ap.alloc(nseg);
  pperm_off_ = ap.alloc(4 * nseg);
  pcnt_off_ = ap.alloc(4 * ((nseg + dev::kVsChunk - 1) / dev::kVsChunk + 1) * (k + 1));
  const int64_t o_in = ap.alloc(4 * static_cast<int64_t>(xin.size()));
  e.ct_off = pair ? ap.alloc(4ll * k * slots * n) : -1;
  const int64_t o_out = ap.alloc(table_bytes(e.Cps));
  const int64_t o_col = ap.alloc(std::max<int64_t>(n, 1));
  const int64_t o_dummy = ap.alloc(2 * static_cast<int64_t>(e.slot_K + 1) * slots);
  const int64_t o_xm = ap.alloc(2 * std::max<int64_t>(static_cast<int64_t>(xm.size()), 1));
  const int64_t o_part = ap.alloc(8 * std::max<int64_t>(1, static_cast<int64_t>(sched_.at(1)[0].nslots)) *
                                  static_cast<int64_t>(e.rooted_smem / (4 * dev::kSpmmWarps * (128 / rl.zw))));
  char* scratch = nullptr;
  std::vector<float> pp(dev::table_floats(e.Cps, n));
  try {
    TCG_CUDA(cudaMalloc(&scratch, std::max<int64_t>(ap.peak, kAlign)));
    arena_ = scratch;
    rooted_parts_ = 1;
    d_partial_ = reinterpret_cast<double*>(scratch + o_part);
    const std::vector<int16_t> dummy = dummy_slots(rl, e.slot_K);
    e.d_slot_acc = reinterpret_cast<int16_t*>(scratch + o_dummy);
    TCG_CUDA(cudaMemcpyAsync(e.d_slot_acc, dummy.data(), 2 * dummy.size(), cudaMemcpyHostToDevice, stream_));
    if (pair) {
      e.d_xmap = reinterpret_cast<int16_t*>(scratch + o_xm);
      TCG_CUDA(cudaMemcpyAsync(e.d_xmap, xm.data(), 2 * xm.size(), cudaMemcpyHostToDevice, stream_));
    }
    uint8_t* dcol = reinterpret_cast<uint8_t*>(scratch + o_col);
    if (n) TCG_CUDA(cudaMemcpyAsync(dcol, lc.data(), n, cudaMemcpyHostToDevice, stream_));
    TCG_CUDA(cudaMemcpyAsync(scratch + o_in, xin.data(), 4 * xin.size(), cudaMemcpyHostToDevice, stream_));
    if (n > 0) {
      bucket_coloring(dcol, dcol, k, nullptr, pair);
      const bool save_ema = rooted_ema_;
      rooted_ema_ = true;  // the input is already in the SpMM's layout
      try {
        rooted_spmm(e, reinterpret_cast<const float*>(scratch + o_in), reinterpret_cast<float*>(scratch + o_out), dcol);
      } catch (...) {
        rooted_ema_ = save_ema;
        throw;
      }
      rooted_ema_ = save_ema;
    }
    TCG_CUDA(cudaStreamSynchronize(stream_));
    copy_sync(pp.data(), scratch + o_out, 4 * pp.size(), cudaMemcpyDeviceToHost);
  } catch (...) {
    arena_ = asave;
    rooted_parts_ = psave;
    d_partial_ = part_save;
    rcol_off_ = o_rc; rcut_off_ = o_cut; lcnt_off_ = o_lc; pseg_off_ = o_seg; pkey_off_ = o_key;
    pperm_off_ = o_perm; pcnt_off_ = o_cnt;
    if (scratch) cudaFree(scratch);
    throw;
  }
  arena_ = asave;
  rooted_parts_ = psave;
  d_partial_ = part_save;
  rcol_off_ = o_rc; rcut_off_ = o_cut; lcnt_off_ = o_lc; pseg_off_ = o_seg; pkey_off_ = o_key;
  pperm_off_ = o_perm; pcnt_off_ = o_cnt;
  cudaFree(scratch);
  tables_valid_ = false;
  // P' storage -> caller order, full C(k, s) columns
  std::fill(y, y + static_cast<int64_t>(nglob_) * C, 0.f);
  std::vector<uint32_t> mask(static_cast<size_t>(C));
  std::vector<int64_t> rel;
  for (int64_t c = 0; c < C; ++c) {
    set_of(k, c, s, cs);
    uint32_t m = 0;
    for (int j = 0; j < s; ++j) m |= 1u << cs[j];
    mask[static_cast<size_t>(c)] = m;
  }
  if (pair) {
    rel.assign(static_cast<size_t>(C) * k, -1);
    for (int64_t c = 0; c < C; ++c) {
      set_of(k, c, s, cs);
      for (int q = 0; q < k; ++q)
        if (!(mask[static_cast<size_t>(c)] >> q & 1u)) {
          int tt[kMaxK];
          for (int j = 0; j < s; ++j) tt[j] = cs[j] > q ? cs[j] - 1 : cs[j];
          rel[static_cast<size_t>(c) * k + q] = index_of(tt, s);
        }
    }
  }
  for (int64_t v = 0; v < n; ++v) {
    const int cv = lc[v];
    for (int64_t c = 0; c < C; ++c) {
      if (mask[static_cast<size_t>(c)] >> cv & 1u) continue;
      const int64_t col = pair ? rl.perm[rel[static_cast<size_t>(c) * k + cv]] : rl.perm[c];
      y[static_cast<int64_t>(perm[v]) * C + c] = pp[dev::panel_offset(e.Cps, n, v, col)];
    }
  }
}

}  // namespace tcg
