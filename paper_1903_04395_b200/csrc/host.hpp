// host.hpp -- host-side subsystems of treecount-b200 (C++17).
//
// The north star assigns these to C++ host code:
//   * CSR construction from an edge list     (graph.hpp:46-95)
//   * template validation + partition plan   (templates.hpp:37-90,174-259)
//   * |Aut(T)|                               (templates.hpp:265-339)
//   * combinadic color index + split tables  (color_index.hpp:20-197)
//   * estimator scaling                      (estimator.hpp:26-33,80-91)
//   * the harness input generators           (synthgen.hpp:40-85)
// Results are identical to the reference's; the algorithms are re-designed
// for throughput (parallel counting-sort CSR build, bitmask sub-templates).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tcg {

// Error classes mirroring the reference's exception types.
struct invalid_argument : std::runtime_error { using std::runtime_error::runtime_error; };
// treecount::parse_error (graph.hpp:18-21): bad graph / template INPUT
struct parse_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct resource_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct cuda_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct nonfinite_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct logic_error : std::runtime_error { using std::runtime_error::runtime_error; };

constexpr int kMaxK = 20;  // color_index.hpp:15

// ---------------------------------------------------------------- MT19937-64
// std::mt19937_64 exactly as ISO C++ [rand.predef] defines it; used by the
// harness generators (rng.hpp wraps the same engine).
struct Mt64 {
  uint64_t x[312];
  int i = 312;
  explicit Mt64(uint64_t seed);
  void twist();
  uint64_t next() {
    if (i >= 312) twist();
    uint64_t z = x[i++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    return z ^ (z >> 43);
  }
  // rng.hpp:21-27
  uint32_t below(uint32_t bound) {
    const uint64_t limit = (UINT64_MAX / bound) * static_cast<uint64_t>(bound);
    uint64_t v = next();
    while (v >= limit) v = next();
    return static_cast<uint32_t>(v % bound);
  }
  // rng.hpp:30
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// -------------------------------------------------------------------- graph
struct Csr {
  int32_t n = 0;
  std::vector<int64_t> row_ptr;  // n+1
  std::vector<int32_t> col;      // nnz, sorted per row
  int64_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
  int32_t max_degree() const;
};

int host_threads();
// fn(begin, end, worker) over [0, total) in static slices on the host threads
void parallel_for(int64_t total, const std::function<void(int64_t, int64_t, int)>& fn);
// graph.hpp:65-95; throws invalid_argument on out-of-range ids.
Csr csr_from_edges(const int32_t* edges, int64_t m, int32_t n_hint);
// validates sorted / loop-free / duplicate-free / in range, and (check_symmetry)
// that every edge appears in both rows (O(nnz log d))
Csr csr_adopt(int32_t n, const int64_t* row_ptr, const int32_t* col, bool check_symmetry = true);
Csr generate_rmat(int scale, int64_t edges, double a, double b, double c, double d,
                  uint64_t seed);
Csr generate_erdos_renyi(int32_t n, double p, uint64_t seed);

// ------------------------------------------------------- color index (k<=20)
struct Binom {
  int64_t c[kMaxK + 1][kMaxK + 1];
  Binom();
  int64_t operator()(int a, int b) const { return (b < 0 || a < 0 || b > a) ? 0 : c[a][b]; }
};
const Binom& binom();
int64_t index_of(const int* colors, int h);                 // color_index.hpp:44-56
void set_of(int k, int64_t index, int h, int* colors);      // color_index.hpp:60-72
// bitmask of an indexed h-set
uint32_t set_mask(int k, int64_t index, int h);

struct SplitTable {  // color_index.hpp:91-101
  int parent_size = 0, active_size = 0, passive_size = 0;
  int32_t parent_cols = 0, active_cols = 0, passive_cols = 0;
  int pairs_per_parent = 0, partners_per_passive = 0;
  std::vector<int32_t> active_index, passive_index;    // [I_s*pairs + p]
  std::vector<int32_t> grouped_parent, grouped_active; // [I_p*partners + q]
};
SplitTable build_split_table(int k, int parent_size, int active_size);  // :103-180

// ------------------------------------------------- rooted-color compression
// A sub-template table M_p[u,S] is zero unless S contains u's own color (the
// root of T_p is mapped to u), so only C(k-1,s-1) of its C(k,s) columns can
// be nonzero: a fraction s/k.  The compressed table keeps, for every vertex,
// just those columns, arranged so the SpMM over it can still accumulate into
// whole output columns:
//   * the C(k,s) sets are partitioned into `groups` groups F_g such that, for
//     every color c, at most `zw` sets of F_g contain c;
//   * compressed panel g of vertex u (zw floats) holds M_p[u,S] for the sets
//     S in F_g that contain color(u), in slot order;
//   * the SpMM output P' is stored GROUP-MAJOR: group g owns the storage
//     columns [fbase[g], fbase[g] + fsize[g]), fbase 8-aligned (32 B sectors),
//     so one pass over compressed panel g produces P' columns F_g complete.
// (B200 design, no reference counterpart: the reference gathers every column.)
struct RootedLayout {
  int k = 0, s = 0;
  int zw = 0;                      // compressed panel width: 8, 16 or 32 floats
  int groups = 0;
  int32_t full_cols = 0;           // C(k,s)
  int32_t store_cols = 0;          // P' storage columns (sum of 8-aligned groups)
  std::vector<int32_t> fsize, fbase;
  std::vector<int32_t> perm;       // full (combinadic) column -> storage column
  std::vector<int32_t> inv;        // storage column -> full column, or -1 (padding)
  std::vector<int16_t> slot_acc;   // [c * groups * zw + g * zw + t] -> index in F_g, or -1
  std::vector<int32_t> slot_col;   // same slots -> full column, or -1
};
RootedLayout build_rooted_layout(int k, int s);

// ----------------------------------------------------------------- template
struct Plan {  // templates.hpp:143-170
  int k = 0, root = 0, num_nodes = 0;
  std::vector<int> size, node_root, active, passive, parent, dp_order;
  std::vector<uint32_t> vertices;  // bitmask per node
  bool is_leaf(int id) const { return size[id] == 1; }
  int full_node() const { return dp_order.back(); }
};
struct Template {
  int k = 0, root = 0;
  std::vector<std::pair<int, int>> edges;
  std::vector<uint32_t> adj;  // neighbour bitmask per template vertex
};
// make_template (templates.hpp:80-90): validate, root<0 -> default_root
Template make_template(int k, const int32_t* edges, int root);
Plan partition(const Template& t);                          // templates.hpp:249-259
uint64_t automorphism_count(const Template& t);             // templates.hpp:326-339
int64_t estimate_bytes(const Plan& plan, int64_t n);        // count_table.hpp:113-133
double colorful_probability(int k);                         // estimator.hpp:29-33

}  // namespace tcg
