// Internal interface of the lowering (csrc/lower*.cpp): the group context,
// the per-template analyses and plans, and the code-emission helpers they
// share.  Not part of the C ABI.
#pragma once

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "emit.hpp"
#include "lower.hpp"

namespace sfx {
namespace lw {

constexpr int kNumSMs = 148;

struct Ctx {
  const Graph& g;
  const Program& p;
  std::vector<int> topo;
  std::vector<int> reduces;
  std::vector<int> dots;  // BatchMatMul members (fuse_dot groups): literal tier only
  std::map<int, bool> dep;
  bool wide = false;
  bool peer = false;  // column sums combine across ranks (opts.cross_rank)
  std::string name;
  Ctx(const Graph& g_, const Program& p_) : g(g_), p(p_) {}
};

int64_t prod(const std::vector<int64_t>& d, size_t b, size_t e);
std::string sanitize(const std::string& s);
bool degenerate_reduce(const Graph& g, const Node& n);
// Templates divide by reduction results through a reciprocal (Emitter::
// rcp_reduced_divisors); SFX_EXACT_DIV=1 keeps the IEEE division (A/B).
bool rcp_divisors();
Ctx make_ctx(const Graph& g, const Program& p);

// ---- kernel scaffolding (lower_analyze.cpp) ----
std::string signature(const Ctx& c, Emitter& em, const std::string& entry, int block, int min_blocks = 0,
                      bool stream = false);
void fill_common(const Ctx& c, KernelSource& ks);
std::string assemble(const std::string& sig, const Code& body);
void emit_stream_gate(Code& body, const std::string& e0, int64_t cta_elems, int64_t total);
void emit_stream_done(Code& body, const std::string& e0);
int64_t gcd64(int64_t a, int64_t b);
int root_slot(const Ctx& c, int node);
int prefix_split(const std::vector<int64_t>& dims, int64_t R);
std::vector<Ix> rowcol_comps(Emitter& em, const std::vector<int64_t>& dims, int64_t R, int64_t C,
                             const Ix& row, const Ix& col);
bool bcast_is_reshape(const Node& m);
bool transpose_is_reshape(const Node& m);

// ---- analyses (lower_analyze.cpp) ----
struct RowPlan {
  int64_t R = 0, C = 0;
  std::map<int, int> cls;
  std::map<int, int> level;
  int max_level = 0;
};
bool analyze_row(const Ctx& c, RowPlan* rp, std::string* why);
struct ColPlan {
  int64_t O = 0, R = 0, I = 0;  // [outer | reduced | inner] of every reduce operand
};
bool analyze_col(const Ctx& c, ColPlan* cp, std::string* why);
// Column reductions over one contiguous block of dims ([outer | reduced |
// inner], like COL) whose results are broadcast back over the reduced dims and
// combined with the elements again — batch-norm's mean / var / normalise, the
// pattern the reference plans as one group with a Column schedule (one block
// per column).  Classes: FULL ([O, R, I] elements) and COLV ([O, I] columns).
struct ColBcPlan {
  int64_t O = 0, R = 0, I = 0;
  std::map<int, int> level;
  int max_level = 0;
};
bool analyze_colbc(const Ctx& c, ColBcPlan* bp, std::string* why);
// Channel statistics broadcast back with the reduced dims on BOTH sides of the
// kept block — [A | K | B], reduce over A and B (batch-norm over NCHW: reduce
// {0, 2, 3}, keep C; the reference plans it as one group of one block).
// Classes: FULL (A·K·B elements) and CHAN (K channels).  f32 sums only.
struct SplitPlan {
  int64_t A = 0, K = 0, B = 0;
  std::map<int, int> level;
  int max_level = 0;
};
bool analyze_colbc_split(const Ctx& c, SplitPlan* sp, std::string* why);
bool analyze_map(const Ctx& c, std::string* why);

// ---- map + tiled transpose (lower_map.cpp) ----
constexpr int kUnknown = -2;
using DimLabel = std::vector<std::pair<int, int64_t>>;
using Labels = std::vector<DimLabel>;
bool labels_known(const Labels& t);
std::map<int, std::set<Labels>> index_labels(const Ctx& c, int root);
struct TilePlan {
  int a = -1, b = -1;  // root axes: a = innermost (output-coalesced), b = input-innermost
  std::map<int, Emitter::Tile> inputs;  // external -> where axes a and b sit in its index
  std::map<int, Labels> labels;         // external -> its labelling
};
bool analyze_tiled(const Ctx& c, TilePlan* tp);
KernelSource lower_map(const Ctx& c, const sfx_compile_opts& o);
KernelSource lower_map_tiled(const Ctx& c, const TilePlan& tp, const sfx_compile_opts& o);
KernelSource lower_map_tiled_v4(const Ctx& c, const TilePlan& tp, const sfx_compile_opts& o);

// ---- row templates (lower_row.cpp) ----
int row_tpr(int64_t C, int V, int streams = 1);
KernelSource lower_row(const Ctx& c, const RowPlan& rp, const sfx_compile_opts& o);
KernelSource lower_row_mp(const Ctx& c, const RowPlan& rp, const sfx_compile_opts& o);
KernelSource lower_row_res(const Ctx& c, const RowPlan& rp, const std::set<int>& staged_inputs,
                           const sfx_compile_opts& o);
KernelSource lower_row_pipe(const Ctx& c, const RowPlan& rp, const std::set<int>& staged_inputs,
                            const sfx_compile_opts& o);
void emit_row_body(const Ctx& c, const RowPlan& rp, Emitter& em, Code& body, int TPR, int V, int64_t NCH);
std::set<int> row_local_inputs(const Ctx& c, const RowPlan& rp);
std::set<int> identity_inputs(const Ctx& c, int64_t full);

// ---- column templates (lower_col.cpp) ----
std::vector<Ix> orc_comps(Emitter& em, const std::vector<int64_t>& dims, int64_t O, int64_t R, int64_t I,
                          const Ix& o, const Ix& r, const Ix& i);
KernelSource lower_col(const Ctx& c, const ColPlan& cp, const sfx_compile_opts& o);
KernelSource lower_colbc(const Ctx& c, const ColBcPlan& bp, const sfx_compile_opts& o);
KernelSource lower_colbc_split(const Ctx& c, const SplitPlan& sp, const sfx_compile_opts& o);
// A second-level sum of squared deviations from the broadcast first-level
// total, b = Σ (u - m)², m = A or scale(A), A = Σ u over the same dims
// (batch-norm's / LayerNorm's var.sum over d2 = d * d, d = x - mean_b).  Such a
// b needs no pass of its own: shifted sums S1 = Σ (u - K), S2 = Σ (u - K)² with
// K = u at reduced index 0 (the same K for every partial of that reduction) fold in A's
// pass, and A = N·K + S1, b = S2 - 2δ·S1 + N·δ², δ = m - K with m the fp32
// mean the graph computes from A (all in fp64: b is the sum of (u - m)² around
// that fp32 mean, the rounding of each d and d² left out — a reduction-order
// class difference within the fp64-checked tolerance).  Empty unless every
// level-2 reduce is such a b (max_level 2, no cross-rank combine);
// SFX_COLBC_TWO_PASS=1 disables it.
struct Var2 {
  int a = -1, b = -1, u = -1, mb = -1;
};
std::vector<Var2> find_var2(const Ctx& c, const std::map<int, int>& level, int max_level);

// ---- literal tier (lower_literal.cpp) ----
KernelSource lower_literal(const Ctx& c);

}  // namespace lw
}  // namespace sfx
