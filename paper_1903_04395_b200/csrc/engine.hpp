// engine.hpp -- the per-GPU DP engine behind the C ABI (include/tcg.h).
//
// Drop-in for the reference's vectorized engine: IterationRun::run
// (engines.hpp:106-132) + vectorized_node (224-268), with the count tables
// resident in HBM as fp32 panels (layout.hpp) and the root in fp64.
// Device memory for one coloring is planned once per (graph, template) by
// simulating the reference's liveness rule (engines.hpp:149-151,
// count_table.hpp:113-133) over a single arena, so a coloring performs no
// allocation and its launch sequence is fixed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tcg.h"
#include "host.hpp"
#include "layout.hpp"

namespace tcg {

// host-only self-check of the ema_rtv_blocked task layout (engine.cu); throws on an inconsistency
void rtv_task_layout_check(int k, int s, int a, int V, int64_t info[6]);

struct NodeExec {
  int id = -1, a = -1, p = -1;
  int size = 0, sa = 0, sp = 0;
  int32_t Cs = 0, Ca = 0, Cp = 0;
  int pairs = 0;
  bool a_leaf = false, p_leaf = false, root = false;
  int2* d_split = nullptr;   // by-parent (I_a, I_p) pairs, [Cs * pairs]
  int32_t* d_drop = nullptr; // active leaf: [Cs * k] column of S minus c, or -1
  uint32_t* d_packed = nullptr;  // (I_a | I_p << 16) when both fit in 16 bits
  // register-blocked eMA (kernels.cuh ema_blocked): output groups + blocks
  bool blocked = false;
  void* d_groups = nullptr;      // dev::GroupDesc[ngroups], sorted by work
  void* d_blocks = nullptr;      // dev::BlockDesc[]
  int ngroups = 0;
  int64_t out_off = -1;      // arena offset of M_s (root: fp64 n)
  int64_t pp_off = -1;       // arena offset of P' (passive internal child)
  size_t ema_smem = 0;
  bool ema_staged = true;
  bool vtx = false;              // vertex-per-CTA eMA (32-vertex tile does not fit smem)
  size_t vtx_smem = 0;
  // rooted-color compressed SpMM (host.hpp RootedLayout): the passive child's
  // table is compressed to `rl_groups` panels of rl_zw slots, P' is stored
  // group-major with Cps columns (== Cp when not rooted)
  bool rooted = false;
  int32_t Cps = 0;
  int rl_zw = 0, rl_groups = 0;
  std::vector<int32_t> rl_fbase, rl_fsize, rl_perm;
  int16_t* d_slot_acc = nullptr;  // [K + 1][groups * zw], unused slots -> the group's dummy (spmm_rooted)
  int slot_K = 0;                 // colors of the slot table: k, or k - 1 (pair layout)
  int32_t* d_slot_col = nullptr;  // [k][groups * zw]
  int32_t* d_pinv = nullptr;      // [Cps] storage column -> combinadic column (blocked eMA staging)
  int64_t ct_off = -1;            // arena offset of the compressed passive table (pair: its copies)
  size_t rooted_smem = 0;         // spmm_rooted dynamic smem
  // pair layout (host.hpp build_pair_layout, rooted eMA only): the rl_*
  // fields, Cps and d_slot_acc then describe the (k-1)-color layout of the
  // sets that miss the ROW's color; the RR passive table is expanded into one
  // copy per row color (pair_expand) and P' is stored relative to c(v)
  bool pair_cand = false, pair = false;
  RootedLayout pr;                // the (k-1)-color layout (candidates)
  int32_t Wx = 0;                 // RR columns of the passive table, C(k-1, sp-1)
  int16_t* d_xmap = nullptr;      // [k][k][groups * zw] copy slot -> RR column, or -1
  std::vector<int16_t> xmap_host;
  // the passive child is an active-leaf node whose table is never written
  // (virt_px): the expansion reads the child's P' through xmap composed with
  // the child's output map (copy slot -> P' storage column)
  int16_t* d_xmap_v = nullptr;
  std::vector<int32_t> cmap_host; // active leaf: [k][Cout] output column -> P' storage column
  bool virt_px = false;
  // rooted eMA (kernels_rt.cuh): same-color vertex tiles of the (k-1)-color
  // problem (s-1, a-1, p); tables stored rooted (RR) or in the parent SpMM's
  // slot layout (RS, passive children)
  int32_t Wa = 0, Wp = 0, Ws = 0; // A columns (RR), staged P rows, relabeled output columns
  int32_t Cout = 0;               // output table columns (Ws for RR, groups * zw for RS)
  int32_t Cpt = 0;                // P' storage columns (hist: k)
  int32_t* d_pmap = nullptr;      // [k][Cpt] P' storage column -> staged row, or -1
  int32_t* d_omap = nullptr;      // [k][Ws] relabeled output column -> slot (RS only)
  int32_t* d_cmap = nullptr;      // active leaf: [k][Cout] output column -> P' storage column
  int32_t* d_imap = nullptr;      // RS: [k][Cout] slot -> relabeled output column, or -1
  std::vector<int32_t> omap;      // host copy (node_table expansion)
  uint32_t* d_rt_packed = nullptr;
  int2* d_rt_split = nullptr;     // root
  int rt_pairs = 0;
  bool rt_blocked = false;
  void* d_rt_groups = nullptr;
  void* d_rt_blocks = nullptr;
  int rt_ngroups = 0;
  size_t rt_smem = 0;
  size_t rt_tma_smem = 0;         // > 0: ema_rt_blocked_tma (raw rows + transposed tile fit one SM)
  size_t rt_pipe_smem = 0;        // > 0: ema_rt_blocked_pipe (two transposed tiles fit one SM)
  bool rt_vtx = false;            // vertex-per-CTA rooted eMA (the 32-vertex tile does not fit smem)
  int rtv_V = 1, rtv_sa = 0, rtv_sp = 0, rtv_h = 6;
  // ema_rtv_blocked tasks (engine.cu build_rtv_tasks): 32 / V same-shape groups per task
  void* d_rtv_tasks = nullptr;        // dev::RtvTask[ntasks]
  int32_t* d_rtv_gout = nullptr;      // [ntasks][32 / V] output column offset of the group, -1 = padding lane
  uint32_t* d_rtv_runs = nullptr;     // pattern runs {i * 16 + j | length << 8}, shared by the tasks of a shape
  uint32_t* d_rtv_blocks = nullptr;   // step-major {a_off | p_off << 16} per (task, block step, group)
  int rtv_ntasks = 0;
  bool rtv_one_cta = false;           // one 896-thread CTA per SM over twice the vertices (very wide rows)
  bool rtv_pleaf = false;         // vertex-per-warp eMA over a leaf passive child (ema_rtv_pleaf)
  uint32_t* d_rtv_drop = nullptr; // [Ws][s-1] {A index of S' minus d | d << 16}
  bool rtv_packed = false;        // d_rtv_drop packed as one uint4 per output (s-1 <= 6, k-1 <= 16)
  // active-leaf node with an unshared rooted SpMM: P' is never materialized --
  // each group's columns go to an n x Ct scratch table and are scattered into
  // the output (RR or RS) right after the group's last part (pstream_copy)
  bool pstream = false;
  int32_t Ct = 0;
  int32_t* d_emap = nullptr;      // [k][Cps] P' storage column -> output column (RS slot / packed q), or -1
  int32_t* d_amap = nullptr;      // packed RR output: [k][Ws] q -> RR column (for its consumer's staging)
  std::vector<int32_t> amap_host;
  int32_t Ca_in = 0;              // storage columns of the active input (Wa, or the virtual child's P' width)
  bool virt = false;              // active-leaf node read only as an active child: its table IS its P',
                                  // staged by the parent through this node's d_pmap (no eMA launch)
  const int32_t* d_amap_in = nullptr;  // this node's ACTIVE input is packed: stage it through this map  // vertices per pass, their smem row strides
  int dup_of = -1;                // exec index of an identical earlier node (table aliased)
  int pp_dup_of = -1;             // exec index of an earlier node with the same P' (SpMM skipped)
};

// SpMM work schedule for one vertex-range part of the gather source.
struct PartSchedule {
  dev::Seg* d_segs = nullptr;   // padded to a multiple of kSegPad
  int64_t nseg_padded = 0;
  int32_t* d_split_rows = nullptr;
  int32_t* d_slot_begin = nullptr;
  int32_t* d_slot_row = nullptr;  // partial slot -> row
  int nsplit_rows = 0, nslots = 0;
  bool owned = true;              // false: buffers live in the engine's graph-prep block
};

// All-gather of equal-size per-rank device buffers (SpMM panels, totals).
struct Transport {
  virtual ~Transport() = default;
  // async() == true: the all-gather is only ENQUEUED on s (stream-ordered);
  // otherwise recv is complete when allgather returns
  virtual bool async() const { return false; }
  virtual void allgather(const void* d_send, size_t bytes, void* d_recv, cudaStream_t s) = 0;
};
void nccl_unique_id(uint8_t* out);   // TCG_NCCL_ID_BYTES bytes
int nccl_version();
std::unique_ptr<Transport> make_nccl_transport(int rank, int world, const uint8_t* id);
std::shared_ptr<void> make_loopback_hub(int world);
std::unique_ptr<Transport> make_loopback_transport(const std::shared_ptr<void>& hub, int rank);
int loopback_world(const std::shared_ptr<void>& hub);
std::unique_ptr<Transport> make_device_transport(tcg_allgather_fn fn, void* user);
std::unique_ptr<Transport> make_host_transport(tcg_allgather_fn fn, void* user);
void set_host_transport_world(Transport* t, int world);
// contiguous row ranges balanced by deg(v) + avg degree
std::vector<int64_t> shard_bounds(int32_t n, const int64_t* row_ptr, int world);

class Engine {
 public:
  void set_shard(int rank, int world, std::unique_ptr<Transport> t);
  bool sharded() const { return world_ > 1 || static_cast<bool>(tr_); }
  int device() const { return cfg_.device; }
  int32_t n_global() const { return nglob_; }
  explicit Engine(const tcg_config& cfg, cudaStream_t shared_stream = nullptr);
  ~Engine();

  void set_graph(const Csr& g);
  // unsharded graph from caller buffers (not copied on the host); validate =
  // check ids / order / loops on the device
  void set_graph_ptrs(int32_t n, const int64_t* row_ptr, const int32_t* col, bool validate, int64_t nnz = -1);
  void set_graph_edges(const int32_t* edges, int64_t m, int32_t n_hint);
  void graph_csr(int32_t* n, int64_t* nnz, int64_t* row_ptr, int32_t* col);
  void set_template(int k, const int32_t* edges, int root);
  int64_t required_bytes() const;
  const Plan& plan() const { return plan_; }
  uint64_t aut() const { return aut_; }
  int32_t n() const { return n_; }

  void coloring(uint64_t seed, uint8_t* host_colors);
  double run_coloring(uint64_t seed, const uint8_t* host_colors, double* per_vertex,
                      tcg_node_stats* stats);
  void estimate(uint64_t seed, int iterations, double* totals, double* est, double* se,
                double* per_vertex_est);
  void node_table(int node_id, int which, double* out);
  void node_table_internal(int node_id, int which, double* out, const std::vector<uint8_t>& colors);
  void spmm_host(const float* x, int cols, float* y);
  void spmm_rooted_host(int k, int s, bool pair, const uint8_t* colors, const float* x, float* y);
  void set_rejection_limit(uint64_t limit) { limit_override_ = limit; }
  int64_t launches() const { return launches_; }
  void time_colorings(uint64_t seed, int count, bool per_kernel, double* totals, tcg_timing* out);

 private:
  void require_ready() const;
  void release_graph();
  void release_template();
  void plan_arena();
  void plan_arena_once(bool allow_stream);
  void ensure_arena();
  void ensure_colors(int64_t bytes);
  void gen_colors(const uint64_t* seeds, int count, uint8_t* d_out);
  // one DP over d_colors; total written to d_total (device), optional root accumulation
  void run_dp(const uint8_t* d_colors, double* d_total, double* d_root_acc,
              tcg_node_stats* stats);
  void spmm(const float* X, float* Y, int64_t cols);
  void hist(const uint8_t* d_colors, float* H);
  float* table_ptr(int64_t off) const { return reinterpret_cast<float*>(arena_ + off); }
  int64_t table_bytes(int64_t cols) const { return 4 * dev::table_floats(cols, n_); }

  // batched colorings: B colorings of a small graph as one DP
  // over the B-fold disjoint union, on a second engine sharing this stream
  struct Batch {
    int B;
    std::unique_ptr<Engine> eng;
    uint64_t tpl_gen, graph_gen;
  };
  std::vector<Batch> batches_;
  int batch_copies_ = 1;             // > 1: this engine holds a union of that many copies
  bool no_relabel_ = false;          // (batch engines: the union keeps its copies contiguous)
  bool own_stream_ = true;
  uint64_t graph_gen_ = 0, tpl_gen_ = 0;
  int pick_batch(int count) const;
  int64_t* d_urp_ = nullptr;         // union CSR scratch (kept across graphs)
  int32_t* d_ucol_ = nullptr;
  int64_t urp_cap_ = 0, ucol_cap_ = 0;
  Engine* batch_engine(int B);
  // B colorings (caller order, nglob_ bytes each) -> totals[B], acc (nullable) += per-vertex
  void run_batch(const uint8_t* d_colors, int B, double* d_totals, double* d_acc);

  // per-kernel event pairs recorded by run_dp when prof_ is set
  struct Prof {
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<size_t, size_t>> spmm, ema;
    cudaEvent_t get();
  };
  Prof* prof_ = nullptr;

  tcg_config cfg_{};
  cudaStream_t stream_ = nullptr;
  int64_t launches_ = 0;
  uint64_t limit_override_ = 0;
  int64_t part_bytes_ = 64ll << 20;  // gather-source footprint per full-table SpMM part
  int rooted_part_mb_ = 0;           // > 0: split the rooted SpMM into colour-class parts of part_bytes_

  // sharding: this rank owns global rows [rows_[rank], rows_[rank+1]); tables
  // have n_ = nmax rows (the largest shard; pad rows have no neighbours);
  // gather ids are padded-global: rank * nmax + local row
  int rank_ = 0, world_ = 1;
  std::unique_ptr<Transport> tr_;
  std::vector<int64_t> rows_;
  int32_t nglob_ = -1, nloc_ = -1;
  int32_t nsrc_ = -1;                // rows of a gather source (world * nmax, or n)
  int64_t* d_rows_ = nullptr;        // rows_ on device
  float* d_xfull_ = nullptr;         // all-gathered panel (world * nmax * 32 floats)
  float* d_xfull2_ = nullptr;        // second buffer: async (NCCL) transports prefetch group g+1
  cudaStream_t comm_ = nullptr;      // communication stream of an async transport
  cudaEvent_t ev_in_ = nullptr, ev_g_[2] = {nullptr, nullptr}, ev_u_[2] = {nullptr, nullptr};
  void ensure_comm();
  uint8_t* d_colors_pad_ = nullptr;  // colors in padded-global order
  double* d_gather_ = nullptr;       // small all-gather scratch (totals)
  void gather_colors(const uint8_t* d_colors);
  void finish_shard_totals(double* totals, int count);  // host: sum over ranks in order
  void gather_per_vertex(const double* d_local, double* host_global);
  // blocking copy ordered on stream_ (stream_ is non-blocking: a plain
  // cudaMemcpy on the legacy stream would not wait for it)
  void copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind);

  // graph
  int32_t n_ = -1;
  int64_t nnz_ = 0;
  int64_t* d_row_ptr_ = nullptr;
  int32_t* d_col_ = nullptr;
  // graph buffers are kept across set_graph calls that fit them (e2e: a new
  // CSR per call without cudaFree/cudaMalloc of ~1 GB); freed by ~Engine
  int64_t row_ptr_cap_ = 0, col_cap_ = 0;
  double* d_est_acc_ = nullptr;      // estimate(): per-vertex fp64 accumulator (n)
  double* d_est_tot_ = nullptr;      // estimate(): totals (iterations)
  int64_t est_acc_cap_ = 0, est_tot_cap_ = 0;
  void free_graph_buffers();
  // part count -> that many part schedules; [1] holds whole rows (also the
  // one-hot histogram's schedule)
  std::map<int, std::vector<PartSchedule>> sched_;
  int parts_for_width(int zw) const;
  void ensure_schedules(int parts);
  void finish_graph(const int64_t* row_ptr, const int32_t* col, bool validate);
  std::vector<int64_t> host_row_ptr_;
  std::vector<int32_t> host_col_;    // only when part schedules are needed (or sharded)
  int max_slots_ = 0;
  int32_t* d_row_order_ = nullptr;   // rows by degree, descending (color_bucket)
  int32_t nlong_ = 0;                // rows of degree > dev::kBucketLong (a prefix of row order)
  int32_t nsmall_ = 0;               // first row (in row order) of degree <= dev::kBucketSmall
  int4* d_lchunks_ = nullptr;        // hub-row chunks {row, begin, end, index in row}
  int32_t* d_lfirst_ = nullptr;      // first chunk of each hub row (nlong_ + 1)
  int32_t nlchunks_ = 0;
  // device-built whole-row schedule + degree order (kernels_graph.cuh): one
  // block reused across set_graph calls of the same (or smaller) size
  char* gp_buf_ = nullptr;
  int64_t gp_n_cap_ = -1, gp_nnz_cap_ = -1;
  void* gp_tmp_ = nullptr;
  size_t gp_tmp_cap_ = 0;
  void prep_graph_device();
  void* cub_tmp(size_t bytes);
  // degree-aware relabeling + isolated-vertex compaction (SURVEY 8(f)4,
  // kernels_graph.cuh): internal row i = caller vertex perm[i]; n_ = rows with
  // a neighbour.  Colors are permuted per coloring, per-vertex results
  // scattered back; the caller never sees internal ids.
  bool relabeled_ = false, rows_sorted_ = true;
  void relabel_device();
  void sort_rows();
  int32_t* d_perm_ = nullptr;        // internal row -> caller vertex (n_ live rows)
  int32_t* d_inv_ = nullptr;         // caller vertex -> internal row, or -1 (isolated)
  int64_t perm_cap_ = 0, inv_cap_ = 0;
  int64_t* d_rp2_ = nullptr;         // relabel scratch: new row_ptr (swapped into d_row_ptr_)
  int32_t* d_col2_ = nullptr;        // relabel scratch: new col (before the per-row sort)
  int64_t rp2_cap_ = 0, col2_cap_ = 0;
  char* rl_buf_ = nullptr;           // relabel scratch: keys, ids, degrees, counter
  int64_t rl_cap_ = -1;
  uint8_t* d_colors_rl_ = nullptr;   // one coloring in internal row order
  int64_t colors_rl_cap_ = 0;
  double* d_pv_out_ = nullptr;       // per-vertex results in caller order (nglob_)
  int64_t pv_out_cap_ = 0;
  std::vector<int32_t> host_perm() ;  // d_perm_ on the host (inspection paths)
  // per-vertex fp64 values of the internal rows -> caller order on the host
  void unpermute_to_host(const double* d_internal, double* host);
  int64_t lcnt_off_ = -1;            // per-coloring chunk color counts [chunks][32]
  int* d_counter_ = nullptr;

  // template / plan
  bool have_template_ = false;
  Template tpl_;
  Plan plan_;
  uint64_t aut_ = 1;
  std::vector<NodeExec> exec_;     // internal nodes in dp order
  bool need_hist_ = false;

  // arena + per-coloring buffers
  int64_t arena_bytes_ = 0;
  int64_t hist_off_ = -1;
  bool need_rooted_ = false;         // some node uses the rooted-compressed SpMM
  bool need_pair_ = false;           // some node uses the pair layout: per-coloring color-ordered segments
  int64_t pseg_off_ = -1, pkey_off_ = -1, pperm_off_ = -1, pcnt_off_ = -1;
  int rooted_parts_ = 1;             // part count of every rooted SpMM (and of the row bucketing)
  int64_t rcol_off_ = -1;            // per-coloring color-sorted packed CSR
  int64_t rcut_off_ = -1;            // per-coloring part (color class) cuts, n * (parts + 1)
  // Pp: full P' (group-major), or the n x Ct scratch of a streamed node (out = its output table)
  void bucket_coloring(const uint8_t* d_gcolors, const uint8_t* d_colors, int k, float* hf, bool pair);
  void rooted_spmm(const NodeExec& e, const float* M, float* Pp, const uint8_t* d_colors, float* out = nullptr);
  bool rooted_ema_ = false;          // every table rooted; eMA on same-color vertex tiles
  int max_tiles_ = 0;                // ceil(n / 32) + k
  int num_sms_ = 148;
  int max_smem_ = 0;
  const uint8_t* d_colors_rt_ = nullptr;  // this context's row colors during run_dp
  int64_t vs_off_ = -1, tiles_off_ = -1, vcnt_off_ = -1;  // per-coloring vertex sort
  void setup_rooted_ema(int max_smem);
  void launch_rt_ema(const NodeExec& e, const float* A, const float* P, double* d_root_acc);
  std::vector<int64_t> table_off_;   // per node id: arena offset of its table (internal)
  std::vector<int64_t> pprime_off_;  // per node id: offset of P' computed from it
  char* arena_ = nullptr;
  int64_t arena_alloc_ = 0;
  double* d_partial_ = nullptr;
  int64_t partial_bytes_ = 0, partial_alloc_ = 0;
  double* d_tile_tot_ = nullptr;
  int64_t tile_tot_cap_ = 0;
  void ensure_tile_tot(int64_t count);
  double* d_scalars_ = nullptr;      // [0] total of run_coloring
  uint8_t* d_colors_ = nullptr;      // color batch
  int64_t colors_cap_ = 0;
  uint64_t* d_seeds_ = nullptr;
  // run_coloring(seed) generates the coloring of seed + 1 on a side stream while the DP of seed
  // runs; a following run_coloring(seed + 1) on the same graph/template finds it ready (the
  // 1.3 ms single-CTA MT19937-64 stream of an n = 1M coloring leaves the critical path)
  struct NextColoring {
    cudaStream_t stream = nullptr;
    cudaEvent_t ready = nullptr;
    uint8_t* d_buf[2] = {nullptr, nullptr};
    uint64_t* d_seed = nullptr;
    int64_t cap = 0;
    int cur = 0;            // d_buf[cur] holds the prefetched coloring
    bool valid = false;
    uint64_t seed = 0, limit = 0;
    int32_t n = 0;
    int k = 0;
  } next_;
  const uint8_t* take_or_generate(uint64_t seed);
  void prefetch_next(uint64_t seed);
  std::vector<uint8_t> last_colors_;
  bool tables_valid_ = false;
};

}  // namespace tcg
