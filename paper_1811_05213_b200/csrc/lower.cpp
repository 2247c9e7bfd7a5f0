#include "lower.hpp"
#include "lower_impl.hpp"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <mutex>
#include <fstream>
#include <cstdlib>
#include <functional>
#include <map>
#include <set>
#include <sstream>

#include "emit.hpp"
#include "jit.hpp"
#include "dyn.hpp"

namespace sfx {

using namespace lw;

std::string choose_strategy(const Graph& g, int pi, std::string* why) {
  const Program& p = g.programs.at(pi);
  if (dot_alone(g, p)) return "dot";
  if (dot_prologue_ok(g, p, nullptr)) return "dotp";
  Ctx c = make_ctx(g, p);
  std::string w;
  if (analyze_map(c, &w)) return "map";
  std::string reasons = "map: " + w;
  RowPlan rp;
  if (analyze_row(c, &rp, &w)) {
    if (rp.C / row_tpr(rp.C, rp.C % 4 == 0 ? 4 : 1) <= 64) return "row";
    w = "row too long for registers";
  }
  reasons += "; row: " + w;
  ColPlan cp;
  if (analyze_col(c, &cp, &w)) return "col";
  reasons += "; col: " + w;
  if (analyze_row(c, &rp, &w)) return "row";  // long rows: clusters / multi-pass (before colbc: measured 7x faster)
  ColBcPlan bp;
  if (analyze_colbc(c, &bp, &w) &&
      (bp.O * bp.I + 127) / 128 <= int64_t{kNumSMs} * 2)  // column tiles fit one co-resident wave
    return "colbc";
  reasons += "; colbc: " + w;
  SplitPlan spl;
  if (analyze_colbc_split(c, &spl, &w)) return "colbc";  // [A | K | B]: channels kept between reduced blocks
  reasons += "; colbc (split): " + w;
  if (why) *why = reasons;
  return "literal";
}

// ---- template parameter cache -------------------------------------------------
//
// Persisted, PerfLibrary-style text (reference tuning.cpp:41-125 stores measured
// schedule costs the same way): one line per group signature
//   signature|rows_per_cta|threads_per_row|items_per_thread|pipe_ctas_per_sm|tuned_us|default_us|source
// where signature = sfx_<template>-<fnv64 of the group's structure> (group_signature).
// tools/autotune.py measures candidate template parameters per group on the
// B200 and writes the winners; lowering with default options looks the group up
// and re-lowers with the recorded parameters.  SFX_TEMPLATE_PARAMS=<file>
// overrides the location, SFX_TEMPLATE_PARAMS=0 disables the cache.
namespace {
struct TunedParams {
  int rows_per_cta = 0, threads_per_row = 0, items_per_thread = 0, pipe_ctas_per_sm = 0;
  std::string note, tuned_us, default_us, source;
};
std::mutex g_tp_mu;  // guards the cache below after loading (template_param_put)
bool g_tp_disabled = false;
std::map<std::string, TunedParams>& template_params() {
  static std::map<std::string, TunedParams> m;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("SFX_TEMPLATE_PARAMS");
    if (e && e[0] == '0' && e[1] == 0) {
      g_tp_disabled = true;
      return;
    }
    std::string path = e ? e : library_dir() + "/template_params.txt";
    std::ifstream in(path);
    std::string line;
    while (std::getline(in, line)) {
      if (line.empty() || line[0] == '#') continue;
      std::vector<std::string> f;
      std::stringstream ss(line);
      std::string x;
      while (std::getline(ss, x, '|')) f.push_back(x);
      if (f.size() < 7) continue;
      TunedParams t;
      t.rows_per_cta = std::atoi(f[1].c_str());
      t.threads_per_row = std::atoi(f[2].c_str());
      t.items_per_thread = std::atoi(f[3].c_str());
      t.pipe_ctas_per_sm = std::atoi(f[4].c_str());
      t.note = "tuned " + f[6] + " -> " + f[5] + " us";
      t.tuned_us = f[5];
      t.default_us = f[6];
      t.source = f.size() > 7 ? f[7] : "";
      m[f[0]] = t;
    }
  });
  return m;
}
bool default_knobs(const sfx_compile_opts& o) {
  return o.rows_per_cta == 0 && o.threads_per_row == 0 && o.items_per_thread == 0 && o.pipe_ctas_per_sm == 0 &&
         o.row_pipeline == 0 && o.pipe_warps == 0 && o.pipe_stages == 0;
}
}  // namespace

KernelSource lower_program_raw(const Graph& g, int pi, const sfx_compile_opts& o);

// The cache key of a group: its template (the entry's sfx_<template> prefix)
// and a hash of what the group computes — members in id order with their
// opcodes, attributes, shapes and dtypes, operands as member / external slot
// references, externals' shapes (splat values inline), roots and the
// cross-rank flag.  Instruction names do not enter, and neither does the
// generated code, so codegen changes keep the recorded parameters (bump
// kTemplateParamsVersion when a template's knobs change meaning).
constexpr const char* kTemplateParamsVersion = "tp2";

std::string group_signature(const Graph& g, int pi, const sfx_compile_opts& o, const std::string& entry) {
  const Program& p = g.programs.at(pi);
  // graph instruction order (members / externals are sorted by name otherwise)
  std::vector<int> members(p.members), externals(p.externals), roots;
  std::sort(members.begin(), members.end());
  std::sort(externals.begin(), externals.end());
  std::map<int, int> local, ext;
  for (size_t i = 0; i < members.size(); ++i) local[members[i]] = static_cast<int>(i);
  for (size_t i = 0; i < externals.size(); ++i) ext[externals[i]] = static_cast<int>(i);
  for (int r : p.roots) roots.push_back(local[r]);
  std::sort(roots.begin(), roots.end());
  std::ostringstream os;
  os << kTemplateParamsVersion << ";x" << (o.cross_rank ? 1 : 0) << ";";
  auto vec = [&](const std::vector<int64_t>& v) {
    os << "[";
    for (int64_t x : v) os << x << ",";
    os << "]";
  };
  for (int e : externals) {
    const Node& n = g.nodes[e];
    os << "E" << n.dtype;
    vec(n.dims);
    if (n.is_splat()) os << "=" << std::hexfloat << n.literal[0] << std::defaultfloat;
    os << ";";
  }
  for (int m : members) {
    const Node& n = g.nodes[m];
    os << "M" << n.op << "." << n.kind << "." << n.dtype << "." << n.reducer << "." << std::hexfloat << n.scalar
       << std::defaultfloat;
    vec(n.dims);
    vec(n.perm);
    vec(n.dim_map);
    vec(n.reduce_dims);
    for (int a : n.operands) os << (local.count(a) ? "m" + std::to_string(local[a]) : "e" + std::to_string(ext[a]));
    os << ";";
  }
  os << "R";
  for (int r : roots) os << r << ",";
  const size_t cut = entry.find('_', 4);
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(fnv1a64(os.str())));
  return entry.substr(0, cut) + "-" + hex;
}

std::string kernel_signature(const Graph& g, int pi, const sfx_compile_opts& o) {
  KernelSource ks = lower_program_raw(g, pi, o);
  return group_signature(g, pi, o, ks.entry);
}

bool template_param_find(const std::string& sig) {
  std::lock_guard<std::mutex> lock(g_tp_mu);
  return template_params().count(sig) > 0;
}

void template_param_put(const std::string& sig, int rows_per_cta, int threads_per_row, int items_per_thread,
                        int pipe_ctas_per_sm, double tuned_us, double default_us, const std::string& source) {
  std::lock_guard<std::mutex> lock(g_tp_mu);
  TunedParams t;
  t.rows_per_cta = rows_per_cta;
  t.threads_per_row = threads_per_row;
  t.items_per_thread = items_per_thread;
  t.pipe_ctas_per_sm = pipe_ctas_per_sm;
  char a[32], b[32];
  std::snprintf(a, sizeof a, "%.2f", tuned_us);
  std::snprintf(b, sizeof b, "%.2f", default_us);
  t.tuned_us = a;
  t.default_us = b;
  t.source = source;
  t.note = "tuned " + t.default_us + " -> " + t.tuned_us + " us";
  template_params()[sig] = t;
}

std::string template_params_text() {
  std::lock_guard<std::mutex> lock(g_tp_mu);
  std::ostringstream os;
  os << "# signature|rows_per_cta|threads_per_row|items_per_thread|pipe_ctas_per_sm|tuned_us|default_us|source\n";
  for (auto& [sig, t] : template_params())
    os << sig << "|" << t.rows_per_cta << "|" << t.threads_per_row << "|" << t.items_per_thread << "|"
       << t.pipe_ctas_per_sm << "|" << t.tuned_us << "|" << t.default_us << "|" << t.source << "\n";
  return os.str();
}

KernelSource lower_program(const Graph& g, int pi, const sfx_compile_opts& o) {
  KernelSource ks = lower_program_raw(g, pi, o);
  const std::string sig = group_signature(g, pi, o, ks.entry);
  if (default_knobs(o)) {
    TunedParams tp;
    bool hit = false;
    {
      std::lock_guard<std::mutex> lock(g_tp_mu);
      auto it = template_params().find(sig);
      if (it != template_params().end()) tp = it->second, hit = true;
    }
    if (hit && (tp.rows_per_cta || tp.threads_per_row || tp.items_per_thread || tp.pipe_ctas_per_sm)) {
      sfx_compile_opts t = o;
      t.rows_per_cta = tp.rows_per_cta;
      t.threads_per_row = tp.threads_per_row;
      t.items_per_thread = tp.items_per_thread;
      t.pipe_ctas_per_sm = tp.pipe_ctas_per_sm;
      ks = lower_program_raw(g, pi, t);
      ks.note += " [template_params: " + tp.note + "]";
    } else if (hit) {
      ks.note += " [template_params: " + tp.note + "]";
    }
  }
  ks.note += " sig=" + sig;
  return ks;
}

// Under cross_rank the graph is one rank's batch shard and dim 0 of every
// tensor is the sharded batch.  A matmul whose contraction axis is dim 0 of an
// operand (traced back through transposes), e.g. dW = X^T * dY, would return a
// per-shard partial sum; no matmul kernel combines across ranks, so such a
// group is refused rather than silently wrong.  (Conservative: a replicated
// weight's dim 0 counts as batch too, like the reductions' rule.)
bool contracts_over_batch(const Graph& g, const Program& p) {
  for (int m : p.members) {
    const Node& n = g.nodes[m];
    if (!is_matmul(n) || n.operands.size() != 2) continue;
    for (int side = 0; side < 2; ++side) {
      int v = n.operands[side];
      int64_t axis = g.nodes[v].rank() - (side == 0 ? 1 : 2);
      while (g.nodes[v].op == SFX_OP_TRANSPOSE && axis >= 0 && axis < static_cast<int64_t>(g.nodes[v].perm.size())) {
        axis = g.nodes[v].perm[axis];  // output axis a reads input axis perm[a] (exec.cpp:172-176)
        v = g.nodes[v].operands[0];
      }
      if (axis == 0) return true;
    }
  }
  return false;
}

KernelSource lower_program_raw(const Graph& g, int pi, const sfx_compile_opts& o) {
  if (pi < 0 || pi >= static_cast<int>(g.programs.size())) throw Error(SFX_ERR_INVALID, "program index out of range");
  const Program& p = g.programs[pi];
  if (o.cross_rank && contracts_over_batch(g, p))
    throw Error(SFX_ERR_UNSUPPORTED, "group " + g.nodes[p.fusion_root].id +
                                         ": a matmul contracts over the sharded dim 0 (cross_rank); only the column "
                                         "templates combine across ranks");
  if (p.barrier && dot_alone(g, p)) return lower_dot(g, p);  // no other lowering for LibraryCall
  Ctx c = make_ctx(g, p);
  std::string why;
  int strat = o.strategy;
  if (o.cross_rank) {
    // the graph is one rank's batch shard: a reduction over dim 0 crosses ranks
    // and only the column template knows how to combine across the peer group
    for (int r : c.reduces)
      for (int64_t d : g.nodes[r].reduce_dims)
        if (d == 0) c.peer = true;
    if (c.peer) {
      // column reductions: the col template; reductions broadcast back
      // (SyncBatchNorm): colbc, whose per-level totals are combined across ranks
      ColPlan cp;
      ColBcPlan bp;
      std::string why2;
      if ((strat == SFX_STRATEGY_AUTO || strat == SFX_STRATEGY_COL) && analyze_col(c, &cp, &why)) {
        strat = SFX_STRATEGY_COL;
      } else if ((strat == SFX_STRATEGY_AUTO || strat == SFX_STRATEGY_COLBC) && analyze_colbc(c, &bp, &why2)) {
        strat = SFX_STRATEGY_COLBC;
      } else {
        throw Error(SFX_ERR_UNSUPPORTED, "group " + c.name +
                                             " reduces over the sharded dim 0 but cannot use the column templates"
                                             " (cross-rank combine): " +
                                             (why.empty() ? "strategy forced" : why + "; " + why2));
      }
    }
  }
  if (strat == SFX_STRATEGY_AUTO) {
    std::string s = choose_strategy(g, pi, &why);
    if (s == "dot") return lower_dot(g, p);
    if (s == "dotp") return lower_dot_prologue(g, p);
    strat = s == "map" ? SFX_STRATEGY_MAP : s == "row" ? SFX_STRATEGY_ROW : s == "col" ? SFX_STRATEGY_COL
            : s == "colbc" ? SFX_STRATEGY_COLBC : SFX_STRATEGY_LITERAL;
  }
  KernelSource ks;
  switch (strat) {
    case SFX_STRATEGY_MAP:
      if (!analyze_map(c, &why)) throw Error(SFX_ERR_UNSUPPORTED, "map template not applicable: " + why);
      {
        TilePlan tp;
        if ((o.items_per_thread == 0 || o.items_per_thread == 1) && analyze_tiled(c, &tp))
          ks = lower_map_tiled(c, tp, o);
        else
          ks = lower_map(c, o);
      }
      break;
    case SFX_STRATEGY_ROW: {
      RowPlan rp;
      if (!analyze_row(c, &rp, &why)) throw Error(SFX_ERR_UNSUPPORTED, "row template not applicable: " + why);
      // Register-resident rows by default.  The TMA-staged pipeline (row-local
      // inputs streamed into shared memory by cp.async.bulk) is available on
      // request: measured on B200 it ties on LayerNorm [8192,1024] and loses
      // 5-25% on softmax / BERT rows (profiles/README.md), because one warp per
      // row already keeps 8-18 independent 128-bit loads in flight.
      std::set<int> staged = row_local_inputs(c, rp);
      bool pipe_ok = !staged.empty() && rp.C % 128 == 0 && rp.C / 32 <= 64 &&
                     4 * 2 * rp.C * 4 * static_cast<int64_t>(staged.size()) <= 200 * 1024 &&
                     o.threads_per_row == 0 && o.rows_per_cta == 0;
      // resident rows: every row of a CTA's range staged at once, one CTA per SM
      const int64_t res_rows = (rp.R + kNumSMs - 1) / kNumSMs;
      bool res_ok = !staged.empty() && rp.C % 128 == 0 && rp.C / 32 <= 64 && o.threads_per_row == 0 &&
                    o.rows_per_cta == 0 && res_rows * (rp.C * 4 * static_cast<int64_t>(staged.size()) + 8) <= 227 * 1024;
      const int Vr = rp.C % 4 == 0 ? 4 : 1;
      if (rp.C / row_tpr(rp.C, Vr) > 64)
        ks = lower_row_mp(c, rp, o);  // longer than 1024 threads x 64 elements
      else if (pipe_ok && o.row_pipeline == 2)
        ks = lower_row_pipe(c, rp, staged, o);
      else if (res_ok && o.row_pipeline == 4)
        ks = lower_row_res(c, rp, staged, o);
      else
        ks = lower_row(c, rp, o);
      break;
    }
    case SFX_STRATEGY_COL: {
      ColPlan cp;
      if (!analyze_col(c, &cp, &why)) throw Error(SFX_ERR_UNSUPPORTED, "col template not applicable: " + why);
      ks = lower_col(c, cp, o);
      break;
    }
    case SFX_STRATEGY_COLBC: {
      ColBcPlan bp;
      SplitPlan spl;
      std::string why_split;
      if (analyze_colbc(c, &bp, &why)) {
        ks = lower_colbc(c, bp, o);
      } else if (!c.peer && analyze_colbc_split(c, &spl, &why_split)) {
        ks = lower_colbc_split(c, spl, o);
      } else {
        throw Error(SFX_ERR_UNSUPPORTED, "colbc template not applicable: " + why + "; split: " + why_split);
      }
      break;
    }
    case SFX_STRATEGY_LITERAL:
      ks = lower_literal(c);
      if (!why.empty()) ks.note += " (" + why + ")";
      break;
    default:
      throw Error(SFX_ERR_INVALID, "unknown strategy");
  }
  return ks;
}

}  // namespace sfx
