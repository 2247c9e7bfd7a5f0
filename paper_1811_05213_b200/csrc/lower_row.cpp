// Row-reduction templates: register-resident rows, TMA-staged rows, long rows (cluster / multi-pass).
#include "lower_impl.hpp"

namespace sfx {
namespace lw {

// ---- ROW ------------------------------------------------------------------------

void emit_row_body(const Ctx& c, const RowPlan& rp, Emitter& em, Code& body, int TPR, int V, int64_t NCH);

// Threads per row: the largest power of two <= 32 dividing the row into
// V-vectors; rows longer than 32 threads x 32 elements span several warps (up
// to a whole CTA) at ~32 elements per thread.
// `streams` = number of [R, C] inputs read per element: rows are widened until
// a thread holds <= 32 streamed values (measured on B200: BERT probs_d / h1
// with 3 streamed inputs gain 4-6% at 2 warps per row; 1-input softmax rows
// are best at one warp).
int row_tpr(int64_t C, int V, int streams) {
  int TPR = 1;
  for (int t = 32; t >= 1; t /= 2)
    if (C % (static_cast<int64_t>(t) * V) == 0) {
      TPR = t;
      break;
    }
  streams = std::max(1, streams);
  while (TPR >= 32 && TPR < 1024 && C / TPR * streams > 32 && C % (static_cast<int64_t>(TPR) * 2 * V) == 0)
    TPR *= 2;
  return TPR;
}

KernelSource lower_row(const Ctx& c, const RowPlan& rp, const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "row";
  ks.entry = "sfx_row_" + c.name;
  fill_common(c, ks);
  const int64_t R = rp.R, C = rp.C;
  int V = (C % 4 == 0) ? 4 : 1;
  int streams = 0;
  for (int n : c.p.inputs)
    if (c.g.nodes[n].numel() == R * C) ++streams;
  int TPR = row_tpr(C, V, streams);
  if (o.threads_per_row > 0) {
    int t = o.threads_per_row;
    if (t > 1024 || (t & (t - 1)) || C % (static_cast<int64_t>(t) * V) != 0)
      throw Error(SFX_ERR_INVALID, "threads_per_row must be a power of two <= 1024 dividing the row");
    TPR = t;
  }
  const int64_t NCH = C / (static_cast<int64_t>(TPR) * V);
  if (NCH * V > 64) throw Error(SFX_ERR_UNSUPPORTED, "row of " + std::to_string(C) + " elements exceeds the register-resident row template");
  const int B = 256;
  int RPC = std::max(1, B / TPR);
  if (o.rows_per_cta > 0 && o.rows_per_cta <= RPC) RPC = o.rows_per_cta;
  const int threads = RPC * TPR;

  // host streaming by row chunks: only when no CTA has out-of-range rows (no
  // thread leaves before the completion barrier)
  const bool stream = o.host_stream && R % RPC == 0 && R > RPC;
  if (stream) {
    ks.stream_R = R;
    ks.stream_C = C;
    ks.stream_cta_elems = int64_t{RPC} * C;
    ks.stream_unit = RPC;
    std::set<int> loc = row_local_inputs(c, rp);
    ks.stream_inputs.assign(loc.begin(), loc.end());
  }
  Emitter em(c.g, c.p, V, c.wide);
  em.rcp_reduced_divisors = rcp_divisors();
  // (pipe_ctas_per_sm doubles as a __launch_bounds__ residency target here)
  std::string sig = signature(c, em, ks.entry, threads, o.pipe_ctas_per_sm, stream);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  if (stream) emit_stream_gate(body, "(long long)blockIdx.x * " + fmt_i(ks.stream_cta_elems), ks.stream_cta_elems, R * C);
  body.line("const int tid = threadIdx.x;");
  body.line("const int lr = tid & " + std::to_string(TPR - 1) + ";");
  if (TPR > 32) {
    body.line("const int rin = tid / " + std::to_string(TPR) + ", wir = (tid & " + std::to_string(TPR - 1) +
              ") >> 5;");
    body.line("const " + it + " row_u = (" + it + ")blockIdx.x * " + std::to_string(RPC) + " + rin;");
    body.line("const bool rvalid = row_u < " + fmt_i(R) + ";");
    body.line("const " + it + " row = rvalid ? row_u : " + fmt_i(R - 1) + ";");
  } else {
    body.line("const " + it + " row = (" + it + ")blockIdx.x * " + std::to_string(RPC) + " + (tid / " +
              std::to_string(TPR) + ");");
    body.line("if (row >= " + fmt_i(R) + ") return;");
  }
  if (TPR >= 32) {
    body.line("const sfx_u32 gmask = 0xffffffffu;");
    body.line("const int gleader = 0;");
  } else if (TPR > 1) {
    if (TPR == 32)
      body.line("const sfx_u32 gmask = 0xffffffffu;");
    else
      body.line("const sfx_u32 gmask = " + std::to_string((1u << TPR) - 1) + "u << ((tid & 31) & " +
                std::to_string(32 - TPR) + ");");
    body.line("const int gleader = (tid & 31) & " + std::to_string(32 - TPR) + ";");
  }
  emit_row_body(c, rp, em, body, TPR, V, NCH);
  if (stream) emit_stream_done(body, "(long long)blockIdx.x * " + fmt_i(ks.stream_cta_elems));
  ks.code = assemble(sig, body);
  ks.block = threads;
  ks.grid_x = (R + RPC - 1) / RPC;
  ks.vector_width = V;
  ks.note = "rows=" + std::to_string(R) + " cols=" + std::to_string(C) + " threads/row=" +
            std::to_string(TPR) + " elems/thread=" + std::to_string(NCH * V) + " levels=" +
            std::to_string(rp.max_level);
  return ks;
}

// Members cached in shared memory between the passes of the cluster variant.
// The final pass (roots) recomputes every inline member it needs from the
// staged slices; a member that the LAST reduction pass already computes (it
// lies under that pass's reduction operands) and whose expression holds an
// expensive op (exp, log, div, pow, tanh, sqrt, rsqrt: ir.cpp's set, the
// reference's `ir.cpp:32-45`) is instead written over a staged input's slice
// in that pass, when the final pass no longer reads that input, and loaded
// back in the final pass (softmax: e = exp(x - max) replaces x, so y = e / sum
// costs one shared-memory load instead of a second exp).  The values are the
// same bits either way.  Only for groups whose [R, C] values are all read at
// the thread's own element (elementwise and reshape-like edges): every thread
// then overwrites only slice elements it alone reads.  Returns member ->
// staged input whose slice it takes.
std::map<int, int> plan_row_cache(const Ctx& c, const RowPlan& rp, const std::vector<int>& staged) {
  const Graph& g = c.g;
  const int64_t RC = rp.R * rp.C;
  std::map<int, int> none;
  if (rp.max_level < 1 || staged.empty()) return none;
  bool ok = true;
  std::set<int> seen;
  std::function<void(int)> check = [&](int n) {
    if (!c.p.is_member(n) || !seen.insert(n).second) return;
    const Node& m = g.nodes[n];
    if (m.numel() == RC) {
      switch (m.op) {
        case SFX_OP_ELEMENTWISE: case SFX_OP_RESHAPE: case SFX_OP_BITCAST: case SFX_OP_BROADCAST:
          break;
        case SFX_OP_TRANSPOSE:
          if (!transpose_is_reshape(m)) ok = false;
          break;
        case SFX_OP_REDUCE:
          if (!degenerate_reduce(g, m)) ok = false;
          break;
        default:
          ok = false;
      }
    }
    for (int o : m.operands) check(o);
  };
  for (int r : c.p.roots) check(r);
  if (!ok) return none;
  // [R, C] members the last reduction pass computes
  std::set<int> avail;
  std::function<void(int)> under = [&](int n) {
    if (!c.p.is_member(n) || avail.count(n)) return;
    const Node& m = g.nodes[n];
    if (m.op == SFX_OP_REDUCE && !degenerate_reduce(g, m)) return;
    if (m.numel() == RC) avail.insert(n);
    for (int o : m.operands) under(o);
  };
  for (int r : c.reduces)
    if (rp.level.at(r) == rp.max_level) under(g.nodes[r].operands[0]);
  std::map<int, bool> exp_memo;
  std::function<bool(int)> costly = [&](int n) -> bool {
    if (!c.p.is_member(n)) return false;
    auto f = exp_memo.find(n);
    if (f != exp_memo.end()) return f->second;
    const Node& m = g.nodes[n];
    bool r = false;
    if (!(m.op == SFX_OP_REDUCE && !degenerate_reduce(g, m))) {
      r = m.op == SFX_OP_ELEMENTWISE && m.kind >= SFX_EW_EXP;
      for (int o : m.operands) r = r || costly(o);
    }
    return exp_memo[n] = r;
  };
  // the final pass's cut: cached members and the staged inputs still read
  std::set<int> cuts, needs, walked;
  std::function<void(int)> walk = [&](int n) {
    if (!walked.insert(n).second) return;
    if (!c.p.is_member(n)) {
      if (std::find(staged.begin(), staged.end(), n) != staged.end()) needs.insert(n);
      return;
    }
    const Node& m = g.nodes[n];
    if (m.op == SFX_OP_REDUCE && !degenerate_reduce(g, m)) return;
    if (avail.count(n) && m.dtype == SFX_F32 && costly(n)) {
      cuts.insert(n);
      return;
    }
    for (int o : m.operands) walk(o);
  };
  for (int r : c.p.roots) walk(r);
  std::vector<int> freed;
  for (int s : staged)
    if (!needs.count(s)) freed.push_back(s);
  if (cuts.empty() || cuts.size() > freed.size()) return none;
  std::map<int, int> out;
  size_t k = 0;
  for (int m : cuts) out[m] = freed[k++];
  return out;
}

// Rows too long to hold in registers (more than 1024 threads x 64 elements,
// e.g. softmax / LayerNorm over 128K columns).
//
// Cluster variant (default when the row's row-local f32 inputs fit the shared
// memory of a thread-block cluster of <= 8 CTAs): one cluster per row, CTA q
// of the cluster owns columns [q*SL, (q+1)*SL).  At entry each CTA has the TMA
// engine copy its slice of every row-local input into shared memory
// (cp.async.bulk + mbarrier); every reduction level is then a pass over shared
// memory, a CTA combine, and a cluster combine through distributed shared
// memory (each CTA publishes its partial, barrier.cluster, every CTA folds the
// CS partials in rank order via ld.shared::cluster — identical results in all
// CTAs); the final pass writes the roots.  HBM sees each input byte once.
//
// Plain variant (inputs too large for a cluster, odd widths): one CTA per row,
// one pass over the row per level plus a final pass, re-reading the row's
// inputs (mostly from L2).  f32 sums accumulate in fp64 per thread.
KernelSource lower_row_mp(const Ctx& c, const RowPlan& rp_in, const sfx_compile_opts& o) {
  KernelSource ks;
  // second moments folded in the first-level pass (find_var2): LayerNorm's
  // variance needs no slice pass and no cluster combine of its own
  const std::vector<Var2> var2 = find_var2(c, rp_in.level, rp_in.max_level);
  RowPlan rp = rp_in;
  std::map<int, const Var2*> var2_a, var2_b;
  for (const Var2& q : var2) {
    rp.level[q.b] = rp.level.at(q.a);
    var2_a[q.a] = &q;
    var2_b[q.b] = &q;
  }
  if (!var2.empty()) rp.max_level = 1;
  ks.strategy = "row";
  fill_common(c, ks);
  const int64_t R = rp.R, C = rp.C;
  const int V = (C % 4 == 0) ? 4 : 1;
  std::set<int> loc = row_local_inputs(c, rp);
  std::vector<int> staged(loc.begin(), loc.end());
  int CS = 1;
  if (V == 4 && !staged.empty() && o.row_pipeline != 1) {  // row_pipeline=1: plain multi-pass (A/B)
    const int64_t bytes = C * 4 * static_cast<int64_t>(staged.size());
    // (pipe_stages doubles as the largest cluster size to consider: 16 is the
    // non-portable maximum)
    // (pipe_stages = 16 / 8 forces the non-portable 16-CTA cluster on / off)
    const int cs_max = o.pipe_stages == 8 ? 8 : 16;
    const int64_t slice_max = o.pipe_stages == 16 ? 32 * 1024 : 64 * 1024;
    int cs = 2;
    while (cs < cs_max && bytes / cs > slice_max) cs *= 2;
    // <= 64 KB of slices per CTA keeps 3 CTAs per SM, so one CTA's TMA load
    // overlaps another's passes; measured: 128 KB slices (1 CTA/SM) lose to
    // the plain multi-pass variant (softmax [256,262144]: 232 vs 185 us)
    if (bytes / cs <= slice_max && C % (int64_t{cs} * V) == 0) CS = cs;
  }
  if (CS == 1) staged.clear();
  ks.entry = (CS > 1 ? "sfx_rowcl_" : "sfx_rowmp_") + c.name;
  int B = CS > 1 ? 512 : 1024;
  if (o.threads_per_row > 0) {
    if (o.threads_per_row % 32 || o.threads_per_row > 1024)
      throw Error(SFX_ERR_INVALID, "threads_per_row must be a multiple of 32 <= 1024 for long rows");
    B = o.threads_per_row;
  }
  const int W = B / 32;
  const int64_t SL = C / CS, SLV = SL / V;  // this CTA's columns / vectors
  // vectors per thread per loop iteration (independent loads in flight)
  const int UR = o.items_per_thread > 0 ? std::min(o.items_per_thread, 16) : 4;
  Emitter em(c.g, c.p, V, c.wide);
  em.rcp_reduced_divisors = rcp_divisors();
  std::string sig = signature(c, em, ks.entry, B);
  if (CS > 1) {
    const std::string gv = "__global__ void ";
    sig.insert(sig.find(gv) + gv.size(), "__cluster_dims__(" + std::to_string(CS) + ", 1, 1) ");
  }
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  body.line("const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;");
  const int64_t slice_bytes = SL * 4;
  const int64_t stage_bytes = slice_bytes * static_cast<int64_t>(staged.size());
  // persistent clusters (row_pipeline=3): NCL clusters loop over the rows, each
  // CTA double-buffering its slices (the TMA copy of row i + 2*NCL is issued as
  // soon as row i's stage is free, so loads run under the passes and stores)
  const bool persist = CS > 1 && o.row_pipeline == 3;
  const int64_t NCL = persist ? std::min<int64_t>(R, std::max<int64_t>(1, (kNumSMs * std::max<int64_t>(
                                                                               1, (220 * 1024) / (2 * stage_bytes))) /
                                                                                  CS))
                              : 0;
  auto issue = [&](const std::string& stage, const std::string& r, const std::string& bar) {
    body.line("  sfx_mbar_expect_tx(" + bar + ", " + fmt_i(stage_bytes) + "u);");
    for (size_t k = 0; k < staged.size(); ++k)
      body.line("  sfx_bulk_g2s(sfx_smem + " + stage + " * " + fmt_i(stage_bytes) + " + " +
                fmt_i(static_cast<int64_t>(k) * slice_bytes) + ", " + em.input_ptr.at(staged[k]) + " + (" + r +
                ") * " + fmt_i(C) + " + (" + it + ")q * " + fmt_i(SL) + ", " + fmt_i(slice_bytes) + "u, " + bar + ");");
  };
  // Cluster combine protocol (default): every CTA pushes its partial of each
  // reduction into slot [rank] of every peer's slot array with st.async, which
  // completes the peer's per-level mbarrier, and folds its own slots in rank
  // order once its mbarrier completes — one relaxed cluster barrier at entry
  // (all mbarriers initialised before any push) instead of a release/acquire
  // cluster barrier per level plus one at exit (each a GPU-scope MEMBAR that
  // also waits for the CTA's outstanding stores, and an L1 invalidation).
  // Persistent clusters double-buffer slots and mbarriers by row parity (a
  // peer is at most one row ahead at any level).  SFX_CLUSTER_BARRIER_COMBINE=1:
  // the barrier protocol (A/B).
  const char* cbenv = std::getenv("SFX_CLUSTER_BARRIER_COMBINE");
  const bool push = CS > 1 && rp.max_level > 0 && !(cbenv && cbenv[0] == '1');
  const int NPAR = persist ? 2 : 1;
  std::vector<int64_t> level_bytes(rp.max_level + 1, 0);
  for (int r : c.reduces) {
    const Node& rn = c.g.nodes[r];
    level_bytes[rp.level.at(r)] += CS * ((rn.reducer == SFX_REDUCE_SUM && rn.dtype == SFX_F32) ? 8 : 4);
  }
  auto arm_levels = [&](const std::string& ind) {
    body.line(ind + "for (int b = 0; b < " + std::to_string(rp.max_level * NPAR) + "; ++b) sfx_mbar_init(cbar + b, 1);");
    body.line(ind + "sfx_fence_mbar_init();");
    for (int lv = 1; lv <= rp.max_level; ++lv)
      for (int pp = 0; pp < NPAR; ++pp)
        body.line(ind + "sfx_mbar_expect_tx(cbar + " + std::to_string((lv - 1) * NPAR + pp) + ", " +
                  fmt_i(level_bytes[lv]) + "u);");
  };
  if (push) body.line("__shared__ __align__(8) unsigned long long cbar[" + std::to_string(rp.max_level * NPAR) + "];");
  if (CS > 1 && persist) {
    body.line("const unsigned q = sfx_cluster_rank();");
    body.line("const " + it + " cid = (" + it + ")blockIdx.x / " + std::to_string(CS) + ";");
    body.line("extern __shared__ __align__(128) unsigned char sfx_smem[];");
    body.line("unsigned long long* sbar = (unsigned long long*)(sfx_smem + " + fmt_i(2 * stage_bytes) + ");");
    body.line("if (tid == 0) {");
    body.line("  sfx_mbar_init(sbar, 1);");
    body.line("  sfx_mbar_init(sbar + 1, 1);");
    if (push) arm_levels("  ");
    body.line("  sfx_fence_mbar_init();");
    body.line("  if (cid < " + fmt_i(R) + ") {");
    issue("0", "cid", "sbar");
    body.line("  }");
    body.line("  if (cid + " + fmt_i(NCL) + " < " + fmt_i(R) + ") {");
    issue("1", "cid + " + fmt_i(NCL), "sbar + 1");
    body.line("  }");
    body.line("}");
    body.line("__syncthreads();");
    if (push) {
      body.line("sfx_cluster_arrive_relaxed();");
      body.line("sfx_cluster_wait();");
    }
    body.line("for (int itr = 0;; ++itr) {");
    body.line("const " + it + " row = cid + (" + it + ")itr * " + fmt_i(NCL) + ";");
    body.line("if (row >= " + fmt_i(R) + ") break;");
    body.line("const int stg = itr & 1;");
    body.line("sfx_mbar_wait_bounded(sbar + stg, (unsigned)((itr >> 1) & 1));");
    ks.smem = static_cast<int>(2 * stage_bytes + 16);
  } else if (CS > 1) {
    body.line("const unsigned q = sfx_cluster_rank();");
    body.line("const " + it + " row = (" + it + ")blockIdx.x / " + std::to_string(CS) + ";");
    body.line("extern __shared__ __align__(128) unsigned char sfx_smem[];");
    const int64_t bar_off = stage_bytes;
    body.line("unsigned long long* sbar = (unsigned long long*)(sfx_smem + " + fmt_i(bar_off) + ");");
    body.line("if (tid == 0) {");
    body.line("  sfx_mbar_init(sbar, 1);");
    if (push) arm_levels("  ");
    body.line("  sfx_fence_mbar_init();");
    body.line("  sfx_mbar_expect_tx(sbar, " + fmt_i(bar_off) + "u);");
    for (size_t k = 0; k < staged.size(); ++k)
      body.line("  sfx_bulk_g2s(sfx_smem + " + fmt_i(static_cast<int64_t>(k) * slice_bytes) + ", " +
                em.input_ptr.at(staged[k]) + " + row * " + fmt_i(C) + " + (" + it + ")q * " + fmt_i(SL) + ", " +
                fmt_i(slice_bytes) + "u, sbar);");
    body.line("}");
    body.line("__syncthreads();");
    if (push) body.line("sfx_cluster_arrive_relaxed();");
    body.line("sfx_mbar_wait(sbar, 0);");
    if (push) body.line("sfx_cluster_wait();  // every peer's mbarriers are initialised before the first push");
    ks.smem = static_cast<int>(bar_off + 16);
  } else {
    body.line("const " + it + " row = (" + it + ")blockIdx.x;");
  }
  Ix rowix = em.uni("row");
  // staged slices: element (row, col) of input k at sl_k[col - q*SL]
  std::map<int, std::pair<std::string, std::string>> staged_map;
  if (CS > 1) {
    std::string rb = em.ivar(Emitter::iadd(em.ivar(Emitter::imul("row", C)), em.ivar(Emitter::imul("q", SL))));
    for (size_t k = 0; k < staged.size(); ++k) {
      std::string p = em.fresh("sl");
      body.line("const float* " + p + " = (const float*)(sfx_smem + " + (persist ? "stg * " + fmt_i(stage_bytes) + " + " : "") +
                fmt_i(static_cast<int64_t>(k) * slice_bytes) + ");");
      staged_map[staged[k]] = {p, rb};
    }
    em.staged = staged_map;
  }
  // (row_pipeline=5: recompute instead of caching, A/B)
  const std::map<int, int> cache = CS > 1 && o.row_pipeline != 5 ? plan_row_cache(c, rp, staged) : std::map<int, int>{};
  std::map<int, std::string> reduced;
  em.resolve = [&](int node, const std::vector<Ix>&) -> std::string {
    if (c.g.nodes[node].op != SFX_OP_REDUCE || degenerate_reduce(c.g, c.g.nodes[node])) return "";
    auto f = reduced.find(node);
    if (f == reduced.end()) throw Error(SFX_ERR_INVALID, "internal: reduction used before it is combined");
    return f->second;
  };
  auto fold_of = [&](const Node& rn) {
    return rn.reducer == SFX_REDUCE_SUM ? "sfx_fold_sum" : rn.reducer == SFX_REDUCE_MAX ? "sfx_fold_pmax"
                                                                                         : "sfx_fold_pmin";
  };
  auto acc_type = [&](const Node& rn) -> std::string {
    return (rn.reducer == SFX_REDUCE_SUM && rn.dtype == SFX_F32) ? "double" : ctype(rn.dtype);
  };
  // a loop over this CTA's vectors, UR per iteration (full tiles unguarded so
  // all UR vectors' loads issue together, then the remainder one at a time);
  // `emit(col_var)` emits one vector's work
  const std::string vbase = CS > 1 ? "(" + it + ")q * " + fmt_i(SLV) + " + " : "";
  auto row_loop = [&](const std::function<void(const std::string&)>& emit) {
    const std::string j = em.fresh("j");
    body.line(it + " " + j + " = tid;");
    body.line("for (; " + j + " + " + std::to_string((UR - 1) * B) + " < " + fmt_i(SLV) + "; " + j + " += " +
              std::to_string(B * UR) + ") {");
    body.indent++;
    em.push();
    for (int u = 0; u < UR; ++u) {
      const std::string ju = em.fresh("ju");
      body.line("const " + it + " " + ju + " = " + vbase + j + " + " + std::to_string(u * B) + ";");
      emit(em.ivar(Emitter::imul(ju, V)));
    }
    em.pop();
    body.indent--;
    body.line("}");
    body.line("for (; " + j + " < " + fmt_i(SLV) + "; " + j + " += " + std::to_string(B) + ") {");
    body.indent++;
    em.push();
    const std::string jv = em.fresh("jv");
    body.line("const " + it + " " + jv + " = " + vbase + j + ";");
    emit(em.ivar(Emitter::imul(jv, V)));
    em.pop();
    body.indent--;
    body.line("}");
  };
  // K per second-moment pair: u at the row's column 0, from global memory (with
  // a cluster it sits in rank 0's slice only); 0 when not finite
  std::map<int, std::string> shiftK;
  for (const Var2& q : var2) {
    em.push();
    em.staged.clear();
    em.lane = 0;
    const std::string v = em.value(q.u, rowcol_comps(em, c.g.nodes[q.u].dims, R, C, rowix, em.uni("0")));
    const std::string k = em.fresh("shk");
    body.line("const double " + k + " = ((__float_as_uint(" + v + ") & 0x7f800000u) != 0x7f800000u) ? (double)" + v +
              " : 0.0;");
    shiftK[q.a] = k;
    em.staged = staged_map;
    em.pop();
  }
  for (int lv = 1; lv <= rp.max_level; ++lv) {
    std::vector<int> red;
    for (int r : c.reduces)
      if (rp.level.at(r) == lv) red.push_back(r);
    std::vector<std::string> acc(red.size());
    for (size_t k = 0; k < red.size(); ++k) {
      const Node& rn = c.g.nodes[red[k]];
      acc[k] = em.fresh("acc");
      std::string init = rn.reducer == SFX_REDUCE_SUM ? (rn.dtype == SFX_F32 ? "0.0" : "0")
                         : rn.dtype == SFX_F32        ? "sfx_bits_f(0x7fc00000)"
                         : rn.reducer == SFX_REDUCE_MAX ? "(int)0x80000000u" : "0x7fffffff";
      body.line(acc_type(rn) + " " + acc[k] + " = " + init + ";");
    }
    row_loop([&](const std::string& cb) {
      for (int lane = 0; lane < V; ++lane) {
        em.lane = lane;
        Ix col = V == 1 ? em.uni(cb) : em.lane_plus(cb);
        for (size_t k = 0; k < red.size(); ++k) {
          if (var2_b.count(red[k])) continue;  // folded with its first-level sum
          const Node& rn = c.g.nodes[red[k]];
          const Node& in = c.g.nodes[rn.operands[0]];
          std::string v = em.value(rn.operands[0], rowcol_comps(em, in.dims, R, C, rowix, col));
          auto qa = var2_a.find(red[k]);
          if (qa != var2_a.end()) {  // shifted sums S1 (a's accumulator), S2 (b's)
            const size_t kb = std::find(red.begin(), red.end(), qa->second->b) - red.begin();
            const std::string t = em.fresh("sh");
            body.line("const double " + t + " = (double)" + v + " - " + shiftK[red[k]] + ";");
            body.line(acc[k] + " += " + t + ";");
            body.line(acc[kb] + " = fma(" + t + ", " + t + ", " + acc[kb] + ");");
            continue;
          }
          body.line(acc[k] + " = " + fold_of(rn) + "(" + acc[k] + ", " + v + ");");
        }
      }
      if (lv != rp.max_level) return;
      // cached members overwrite their slice element after its last read
      for (const auto& [m, x] : cache) {
        const Node& mn = c.g.nodes[m];
        const auto& slot = staged_map.at(x);
        std::vector<std::string> vals(V);
        Ix L0;
        for (int lane = 0; lane < V; ++lane) {
          em.lane = lane;
          Ix col = V == 1 ? em.uni(cb) : em.lane_plus(cb);
          std::vector<Ix> comps = rowcol_comps(em, mn.dims, R, C, rowix, col);
          vals[lane] = em.value(m, comps);
          if (lane == 0) L0 = em.linearize(comps, mn.dims);
          if (V == 1 || L0.kind != IX_PLUS)
            body.line("((float*)" + slot.first + ")[" + em.linearize(comps, mn.dims).e + " - " + slot.second +
                      "] = " + vals[lane] + ";");
        }
        if (V == 4 && L0.kind == IX_PLUS)
          body.line("sfx_sts4((float*)" + slot.first + " + (" + L0.base + " - " + slot.second + "), " + vals[0] +
                    ", " + vals[1] + ", " + vals[2] + ", " + vals[3] + ");");
      }
    });
    std::vector<std::string> slots(red.size());
    const std::string cb_lv = "cbar + " + std::to_string((lv - 1) * NPAR) + (persist ? " + (itr & 1)" : "");
    for (size_t k = 0; k < red.size(); ++k) {
      const Node& rn = c.g.nodes[red[k]];
      const std::string T = acc_type(rn);
      for (int m = 16; m >= 1; m /= 2)
        body.line(acc[k] + " = " + fold_of(rn) + "(" + acc[k] + ", __shfl_xor_sync(0xffffffffu, " + acc[k] + ", " +
                  std::to_string(m) + "));");
      const std::string sm = em.fresh("rsm");
      body.line("__shared__ " + T + " " + sm + "[" + std::to_string(W) + "];");
      body.line("if (lane == 0) " + sm + "[warp] = " + acc[k] + ";");
      body.line("__syncthreads();");
      body.line(acc[k] + " = " + sm + "[0];");
      body.line("for (int w = 1; w < " + std::to_string(W) + "; ++w) " + acc[k] + " = " + fold_of(rn) + "(" + acc[k] +
                ", " + sm + "[w]);");
      if (push) {
        slots[k] = em.fresh("xs");
        body.line("__shared__ " + T + " " + slots[k] + "[" + std::to_string(NPAR) + "][" + std::to_string(CS) + "];");
        body.line("if (tid == 0)");
        body.line("  for (unsigned r = 0; r < " + std::to_string(CS) + "u; ++r) sfx_dsmem_push(&" + slots[k] + "[" +
                  (persist ? "itr & 1" : "0") + "][q], " + acc[k] + ", " + cb_lv + ", r);");
      } else if (CS > 1) {
        // cluster combine: every CTA folds the CS partials in rank order.  One
        // warp reads them (lane r from rank r, one DSMEM load each) and lane 0
        // folds them in order; the CTA reads the result from local smem (all
        // 512 threads reading every rank's slot over DSMEM cost 12% of the
        // kernel's smem wavefronts in conflicts)
        // Persistent clusters reuse the slot row after row: it is double-buffered
        // by row parity, because with a single cluster barrier per reduction a
        // fast CTA may publish row i+1's partial before a peer's warp 0 has read
        // row i's (two rows ahead needs the peer past row i+1's barrier, i.e.
        // done reading row i)
        const std::string xa = em.fresh("xp"), xr = em.fresh("xr");
        const std::string xp = persist ? xa + "[itr & 1]" : xa;
        body.line("__shared__ " + T + " " + xa + (persist ? "[2]" : "") + ";");
        body.line("__shared__ " + T + " " + xr + ";");
        body.line("if (tid == 0) " + xp + " = " + acc[k] + ";");
        body.line("sfx_cluster_sync();");
        body.line("if (warp == 0) {");
        body.line("  const " + T + " v = lane < " + std::to_string(CS) + " ? sfx_dsmem_ld(&" + xp + ", (unsigned)lane) : " +
                  xp + ";");
        body.line("  " + T + " a = __shfl_sync(0xffffffffu, v, 0);");
        body.line("  for (int r = 1; r < " + std::to_string(CS) + "; ++r) a = " + fold_of(rn) +
                  "(a, __shfl_sync(0xffffffffu, v, r));");
        body.line("  if (lane == 0) " + xr + " = a;");
        body.line("}");
        body.line("__syncthreads();");
        body.line(acc[k] + " = " + xr + ";");
      }
    }
    if (push) {
      body.line("sfx_mbar_wait_bounded(" + cb_lv + ", " + (persist ? "(unsigned)((itr >> 1) & 1)" : "0u") + ");");
      if (persist) body.line("if (tid == 0) sfx_mbar_expect_tx(" + cb_lv + ", " + fmt_i(level_bytes[lv]) + "u);  // rearm for row itr + 2");
    }
    std::vector<size_t> order;  // second moments after the first-level sums they use
    for (size_t k = 0; k < red.size(); ++k)
      if (!var2_b.count(red[k])) order.push_back(k);
    for (size_t k = 0; k < red.size(); ++k)
      if (var2_b.count(red[k])) order.push_back(k);
    std::map<int, std::string> raw;  // fp64 totals as folded (S1 for second-moment first levels)
    for (size_t k : order) {
      const Node& rn = c.g.nodes[red[k]];
      const std::string T = acc_type(rn);
      if (push) {
        const std::string sl = slots[k] + "[" + (persist ? "itr & 1" : "0") + "]";
        body.line(acc[k] + " = " + sl + "[0];");
        body.line("for (int r = 1; r < " + std::to_string(CS) + "; ++r) " + acc[k] + " = " + fold_of(rn) + "(" + acc[k] +
                  ", " + sl + "[r]);");
      }
      std::string fin = acc[k];
      raw[red[k]] = acc[k];
      if (var2_a.count(red[k])) {  // A = N·K + S1
        fin = em.fresh("tot");
        body.line("const double " + fin + " = " + fmt_i(C) + ".0 * " + shiftK[red[k]] + " + " + acc[k] + ";");
      }
      auto qb = var2_b.find(red[k]);
      if (qb != var2_b.end()) {  // b = S2 - 2δ·S1 + N·δ², δ = m - K; a non-finite mean as in Σ (u - m)²
        const Var2& q = *qb->second;
        em.push();
        em.staged.clear();
        em.lane = 0;
        const std::string m = em.value(q.mb, rowcol_comps(em, c.g.nodes[q.mb].dims, R, C, rowix, em.uni("0")));
        em.staged = staged_map;
        em.pop();
        const std::string dl = em.fresh("dl");
        fin = em.fresh("tot");
        body.line("const double " + dl + " = (double)" + m + " - " + shiftK[q.a] + ";");
        body.line("const double " + fin + " = ((__float_as_uint(" + m + ") & 0x7f800000u) != 0x7f800000u) ? " + acc[k] +
                  " - 2.0 * " + dl + " * " + raw[q.a] + " + " + fmt_i(C) + ".0 * " + dl + " * " + dl + " : (" + m +
                  " != " + m + " || !(fabs(" + raw[q.a] + ") <= 1.7976931348623157e308)) ? (double)(" + m + " - " + m +
                  ") : (double)(" + m + " * " + m + ");");
      }
      if (T == "double") {
        const std::string d = fin;
        fin = em.fresh("red");
        body.line("const float " + fin + " = (float)" + d + ";");
      }
      if (rn.reducer != SFX_REDUCE_SUM && rn.dtype == SFX_F32) {
        // the sequential fold's first element: the row's element 0, read from
        // global memory (with a cluster it sits in rank 0's slice only)
        em.push();
        em.staged.clear();
        em.lane = 0;
        const Node& in = c.g.nodes[rn.operands[0]];
        std::string f0 = em.value(rn.operands[0], rowcol_comps(em, in.dims, R, C, rowix, em.uni("0")));
        body.line(fin + " = sfx_fold_first(" + f0 + ", " + fin + ");");
        em.staged = staged_map;
        em.pop();
      }
      reduced[red[k]] = fin;
    }
  }
  std::vector<int> full_roots, row_roots;
  for (int r : c.p.roots) (c.g.nodes[r].numel() == R * C ? full_roots : row_roots).push_back(r);
  if (!cache.empty()) {  // the final pass reads the cached members, not the inputs they replaced
    em.staged = staged_map;
    for (const auto& [m, x] : cache) {
      em.staged[m] = staged_map.at(x);
      em.staged.erase(x);
    }
  }
  if (!full_roots.empty())
    row_loop([&](const std::string& cb) {
      std::vector<std::vector<std::string>> vals(full_roots.size(), std::vector<std::string>(V));
      for (int lane = 0; lane < V; ++lane) {
        em.lane = lane;
        Ix col = V == 1 ? em.uni(cb) : em.lane_plus(cb);
        for (size_t k = 0; k < full_roots.size(); ++k)
          vals[k][lane] = em.value(full_roots[k], rowcol_comps(em, c.g.nodes[full_roots[k]].dims, R, C, rowix, col));
      }
      const std::string addr = em.ivar(Emitter::iadd(em.ivar(Emitter::imul("row", C)), cb));
      for (size_t k = 0; k < full_roots.size(); ++k) {
        std::string out = "out" + std::to_string(root_slot(c, full_roots[k]));
        if (V == 4)
          body.line("sfx_st4(" + out + " + " + addr + ", " + vals[k][0] + ", " + vals[k][1] + ", " + vals[k][2] +
                    ", " + vals[k][3] + ");");
        else
          body.line(out + "[" + addr + "] = " + vals[k][0] + ";");
      }
    });
  if (!row_roots.empty()) {
    em.lane = 0;
    em.staged.clear();
    body.line(CS > 1 ? "if (tid == 0 && q == 0) {" : "if (tid == 0) {");
    body.indent++;
    em.push();
    for (int r : row_roots)
      body.line("out" + std::to_string(root_slot(c, r)) + "[row] = " + em.value(r, em.from_linear(rowix, c.g.nodes[r].dims)) +
                ";");
    em.pop();
    body.indent--;
    body.line("}");
  }
  em.staged.clear();
  if (persist) {
    // this stage is free once every thread is past the final pass
    body.line("__syncthreads();");
    body.line("if (tid == 0 && row + " + fmt_i(2 * NCL) + " < " + fmt_i(R) + ") {");
    issue("stg", "row + " + fmt_i(2 * NCL), "sbar + stg");
    body.line("}");
    body.line("}");  // row loop
  }
  if (CS > 1 && !push) body.line("sfx_cluster_sync();  // no CTA leaves while a peer may still read its partials");
  ks.code = assemble(sig, body);
  ks.block = B;
  ks.grid_x = (persist ? NCL : R) * CS;
  ks.cluster = CS;
  ks.vector_width = V;
  // residency cap through dynamic shared memory (plain variant, A/B knob)
  if (CS == 1 && o.pipe_ctas_per_sm > 0) ks.smem = 220 * 1024 / o.pipe_ctas_per_sm;
  if (CS > 1)
    ks.note = "rows=" + std::to_string(R) + " cols=" + std::to_string(C) + " cluster of " + std::to_string(CS) +
              " CTAs x " + std::to_string(B) + " threads per row, " + std::to_string(staged.size()) +
              " input slice(s) of " + std::to_string(slice_bytes) + " B in shared memory (TMA), " + (push ? "DSMEM push combine, " : "DSMEM combine, ") +
              (cache.empty() ? std::string() : std::to_string(cache.size()) + " member(s) cached over input slices, ") + "levels=" +
              std::to_string(rp.max_level) + (persist ? ", persistent: " + std::to_string(NCL) + " clusters, 2 stages" : "") +
              (var2.empty() ? "" : ", " + std::to_string(var2.size()) + " second moment(s) in the first pass");
  else
    ks.note = "rows=" + std::to_string(R) + " cols=" + std::to_string(C) + " one CTA of " + std::to_string(B) +
              " threads per row, multi-pass (" + std::to_string(rp.max_level + (full_roots.empty() ? 0 : 1)) +
              " passes, re-reads from L2) levels=" + std::to_string(rp.max_level) +
              (var2.empty() ? "" : ", " + std::to_string(var2.size()) + " second moment(s) in the first pass");
  return ks;
}

// The row body shared by the register-resident and the TMA-pipelined row
// templates: reduction phases (per-thread fold -> shuffle tree -> broadcast
// back through registers) then the element and row roots.  Expects `row`,
// `lr` (lane within the row group), `gmask`, `gleader` in scope.
void emit_row_body(const Ctx& c, const RowPlan& rp_in, Emitter& em, Code& body, int TPR, int V, int64_t NCH) {
  // SFX_ROW_VAR2=1: the variance folded in the mean's phase here too (fp64
  // shifted sums; one shuffle / shared-memory round instead of two) — A/B
  const char* v2env = std::getenv("SFX_ROW_VAR2");
  const std::vector<Var2> var2 =
      (v2env && v2env[0] == '1') ? find_var2(c, rp_in.level, rp_in.max_level) : std::vector<Var2>{};
  RowPlan rp = rp_in;
  std::map<int, const Var2*> var2_a, var2_b;
  for (const Var2& q : var2) {
    rp.level[q.b] = rp.level.at(q.a);
    var2_a[q.a] = &q;
    var2_b[q.b] = &q;
  }
  if (!var2.empty()) rp.max_level = 1;
  const int64_t R = rp.R, C = rp.C;
  const std::string& it = em.idx_t;
  std::vector<std::string> cb(NCH);
  for (int64_t j = 0; j < NCH; ++j) {
    cb[j] = em.fresh("cb");
    body.line("const " + it + " " + cb[j] + " = lr * " + std::to_string(V) + " + " +
              fmt_i(j * TPR * V) + ";");
  }
  Ix rowix = em.uni("row");
  auto col_ix = [&](int64_t j, int lane) {
    em.lane = lane;
    return V == 1 ? em.uni(cb[j]) : em.lane_plus(cb[j]);
  };
  std::map<int, std::string> reduced;  // reduce node -> combined value
  em.resolve = [&](int node, const std::vector<Ix>&) -> std::string {
    if (c.g.nodes[node].op != SFX_OP_REDUCE || degenerate_reduce(c.g, c.g.nodes[node])) return "";
    auto f = reduced.find(node);
    if (f == reduced.end()) throw Error(SFX_ERR_INVALID, "internal: reduction used before it is combined");
    return f->second;
  };

  std::map<int, std::string> shiftK;
  for (const Var2& q : var2) {
    em.push();
    em.lane = 0;
    const std::string v = em.value(q.u, rowcol_comps(em, c.g.nodes[q.u].dims, R, C, rowix, em.uni("0")));
    const std::string k = em.fresh("shk");
    body.line("const double " + k + " = ((__float_as_uint(" + v + ") & 0x7f800000u) != 0x7f800000u) ? (double)" + v +
              " : 0.0;");
    shiftK[q.a] = k;
    em.pop();
  }
  auto vtype = [&](int r) -> std::string {
    return var2_a.count(r) || var2_b.count(r) ? "double" : ctype(c.g.nodes[r].dtype);
  };
  for (int lv = 1; lv <= rp.max_level; ++lv) {
    std::vector<int> red;
    for (int r : c.reduces)
      if (rp.level.at(r) == lv) red.push_back(r);
    std::vector<std::string> acc(red.size()), first(red.size());
    for (size_t k = 0; k < red.size(); ++k) {
      acc[k] = em.fresh("acc");
      body.line(vtype(red[k]) + " " + acc[k] + (vtype(red[k]) == "double" ? " = 0.0;" : ";"));
    }
    for (int64_t j = 0; j < NCH; ++j)
      for (int lane = 0; lane < V; ++lane) {
        Ix col = col_ix(j, lane);
        for (size_t k = 0; k < red.size(); ++k) {
          if (var2_b.count(red[k])) continue;  // folded with its first-level sum
          const Node& rn = c.g.nodes[red[k]];
          const Node& in = c.g.nodes[rn.operands[0]];
          std::vector<Ix> comps = rowcol_comps(em, in.dims, R, C, rowix, col);
          std::string v = em.value(rn.operands[0], comps);
          auto qa = var2_a.find(red[k]);
          if (qa != var2_a.end()) {
            const size_t kb = std::find(red.begin(), red.end(), qa->second->b) - red.begin();
            const std::string t = em.fresh("sh");
            body.line("const double " + t + " = (double)" + v + " - " + shiftK[red[k]] + ";");
            body.line(acc[k] + " += " + t + ";");
            body.line(acc[kb] + " = fma(" + t + ", " + t + ", " + acc[kb] + ");");
            continue;
          }
          if (j == 0 && lane == 0) {
            body.line(acc[k] + " = " + v + ";");
            first[k] = v;
          } else {
            const char* f = rn.reducer == SFX_REDUCE_SUM ? "sfx_fold_sum"
                            : rn.reducer == SFX_REDUCE_MAX ? "sfx_fold_pmax" : "sfx_fold_pmin";
            body.line(acc[k] + " = " + f + "(" + acc[k] + ", " + v + ");");
          }
        }
      }
    for (size_t k = 0; k < red.size(); ++k) {
      const Node& rn = c.g.nodes[red[k]];
      const char* f = rn.reducer == SFX_REDUCE_SUM ? "sfx_fold_sum"
                      : rn.reducer == SFX_REDUCE_MAX ? "sfx_fold_pmax" : "sfx_fold_pmin";
      for (int m = std::min(TPR, 32) / 2; m >= 1; m /= 2)
        body.line(acc[k] + " = " + f + "(" + acc[k] + ", " +
                  (vtype(red[k]) == "double" ? "__shfl_xor_sync(gmask, " + acc[k] + ", " + std::to_string(m) + ")"
                                             : "sfx_shfl_xor(" + acc[k] + ", " + std::to_string(m) + ", gmask)") +
                  ");");
    }
    const int W = TPR > 32 ? TPR / 32 : 1;  // warps per row
    std::vector<std::string> rsm(red.size()), rfm(red.size());
    if (W > 1) {
      // rows spanning several warps: per-warp partials through shared memory,
      // folded by every thread in warp order (deterministic)
      const int RPC = std::max(1, 256 / TPR);
      for (size_t k = 0; k < red.size(); ++k) {
        const Node& rn = c.g.nodes[red[k]];
        rsm[k] = em.fresh("rsm");
        body.line("__shared__ " + vtype(red[k]) + " " + rsm[k] + "[" + std::to_string(RPC) + "][" +
                  std::to_string(W) + "];");
        body.line("if ((tid & 31) == 0) " + rsm[k] + "[rin][wir] = " + acc[k] + ";");
        if (rn.reducer != SFX_REDUCE_SUM && rn.dtype == SFX_F32) {
          rfm[k] = em.fresh("rfm");
          body.line(std::string("__shared__ float ") + rfm[k] + "[" + std::to_string(RPC) + "];");
          body.line("if (lr == 0) " + rfm[k] + "[rin] = " + first[k] + ";");
        }
      }
      body.line("__syncthreads();");
      for (size_t k = 0; k < red.size(); ++k) {
        const Node& rn = c.g.nodes[red[k]];
        const char* f = rn.reducer == SFX_REDUCE_SUM ? "sfx_fold_sum"
                        : rn.reducer == SFX_REDUCE_MAX ? "sfx_fold_pmax" : "sfx_fold_pmin";
        body.line(acc[k] + " = " + rsm[k] + "[rin][0];");
        for (int w = 1; w < W; ++w)
          body.line(acc[k] + " = " + f + "(" + acc[k] + ", " + rsm[k] + "[rin][" + std::to_string(w) + "]);");
      }
    }
    std::vector<size_t> order;  // second moments after the first-level sums they use
    for (size_t k = 0; k < red.size(); ++k)
      if (!var2_b.count(red[k])) order.push_back(k);
    for (size_t k = 0; k < red.size(); ++k)
      if (var2_b.count(red[k])) order.push_back(k);
    for (size_t k : order) {
      const Node& rn = c.g.nodes[red[k]];
      if (rn.reducer != SFX_REDUCE_SUM && rn.dtype == SFX_F32) {
        std::string f0 = W > 1 ? rfm[k] + "[rin]" : TPR > 1 ? "sfx_shfl(" + first[k] + ", gleader, gmask)" : first[k];
        body.line(acc[k] + " = sfx_fold_first(" + f0 + ", " + acc[k] + ");");
      }
      std::string fin = acc[k];
      if (var2_a.count(red[k])) {  // A = N·K + S1
        fin = em.fresh("red");
        body.line("const float " + fin + " = (float)(" + fmt_i(C) + ".0 * " + shiftK[red[k]] + " + " + acc[k] + ");");
      }
      auto qb = var2_b.find(red[k]);
      if (qb != var2_b.end()) {  // b = S2 - 2δ·S1 + N·δ², δ = m - K; a non-finite mean as in Σ (u - m)²
        const Var2& q = *qb->second;
        size_t ka = std::find(red.begin(), red.end(), q.a) - red.begin();
        em.push();
        em.lane = 0;
        const std::string m = em.value(q.mb, rowcol_comps(em, c.g.nodes[q.mb].dims, R, C, rowix, em.uni("0")));
        em.pop();
        const std::string dl = em.fresh("dl");
        fin = em.fresh("red");
        body.line("const double " + dl + " = (double)" + m + " - " + shiftK[q.a] + ";");
        body.line("const float " + fin + " = (float)(((__float_as_uint(" + m + ") & 0x7f800000u) != 0x7f800000u) ? " +
                  acc[k] + " - 2.0 * " + dl + " * " + acc[ka] + " + " + fmt_i(C) + ".0 * " + dl + " * " + dl + " : (" +
                  m + " != " + m + " || !(fabs(" + acc[ka] + ") <= 1.7976931348623157e308)) ? (double)(" + m + " - " + m +
                  ") : (double)(" + m + " * " + m + "));");
      }
      reduced[red[k]] = fin;
    }
  }

  // final phase: element roots (vectorised stores) and row roots (lane 0)
  std::vector<int> full_roots, row_roots;
  for (int r : c.p.roots) (c.g.nodes[r].numel() == R * C ? full_roots : row_roots).push_back(r);
  const std::string rb = em.ivar(Emitter::imul("row", C));
  for (int64_t j = 0; j < NCH; ++j) {
    std::vector<std::vector<std::string>> vals(full_roots.size(), std::vector<std::string>(V));
    for (int lane = 0; lane < V; ++lane) {
      Ix col = col_ix(j, lane);
      for (size_t k = 0; k < full_roots.size(); ++k)
        vals[k][lane] = em.value(full_roots[k], rowcol_comps(em, c.g.nodes[full_roots[k]].dims, R, C, rowix, col));
    }
    std::string addr = em.ivar(Emitter::iadd(rb, cb[j]));
    // multi-warp rows keep out-of-range rows alive (clamped) for the barriers
    const std::string guard = TPR > 32 ? "if (rvalid) " : "";
    for (size_t k = 0; k < full_roots.size(); ++k) {
      std::string out = "out" + std::to_string(root_slot(c, full_roots[k]));
      if (V == 4)
        body.line(guard + "sfx_st4(" + out + " + " + addr + ", " + vals[k][0] + ", " + vals[k][1] + ", " +
                  vals[k][2] + ", " + vals[k][3] + ");");
      else
        body.line(guard + out + "[" + addr + "] = " + vals[k][0] + ";");
    }
  }
  if (!row_roots.empty()) {
    em.lane = 0;
    body.line(TPR > 32 ? "if (lr == 0 && rvalid) {" : "if (lr == 0) {");
    body.indent++;
    em.push();
    for (int r : row_roots) {
      std::string v = em.value(r, em.from_linear(rowix, c.g.nodes[r].dims));
      body.line("out" + std::to_string(root_slot(c, r)) + "[row] = " + v + ";");
    }
    em.pop();
    body.indent--;
    body.line("}");
  }
}

// External inputs of the row space ([R, C] elements) that are only ever read
// at the current row — safe to stream row by row into shared memory.  An
// operand is row-local when every path to it from a root or a reduction goes
// through row-preserving edges (elementwise, reshape/bitcast, reduce over the
// row, broadcast of a row scalar, reshape-like broadcast/transpose, transpose
// permuting columns only).
std::set<int> row_local_inputs(const Ctx& c, const RowPlan& rp) {
  const Graph& g = c.g;
  const int64_t R = rp.R, C = rp.C;
  std::set<int> local, unsafe;
  std::function<void(int, bool)> walk = [&](int n, bool ok) {
    if (!c.p.is_member(n)) {
      (ok ? local : unsafe).insert(n);
      return;
    }
    const Node& m = g.nodes[n];
    for (int o : m.operands) {
      bool edge = true;
      switch (m.op) {
        case SFX_OP_ELEMENTWISE: case SFX_OP_RESHAPE: case SFX_OP_BITCAST: case SFX_OP_REDUCE:
          break;
        case SFX_OP_BROADCAST: {
          bool prefix = g.nodes[o].numel() == R;
          for (size_t j = 0; prefix && j < m.dim_map.size(); ++j)
            if (m.dim_map[j] != static_cast<int64_t>(j)) prefix = false;
          edge = bcast_is_reshape(m) || prefix;
          break;
        }
        case SFX_OP_TRANSPOSE: {
          int k = prefix_split(m.dims, R);
          edge = transpose_is_reshape(m);
          if (!edge && k >= 0 && prod(m.dims, k, m.dims.size()) == C) {
            edge = true;
            for (int i = 0; i < k; ++i)
              if (m.perm[i] != i) edge = false;
          }
          break;
        }
        default:
          edge = false;
      }
      walk(o, ok && edge);
    }
  };
  for (int r : c.p.roots) walk(r, true);
  std::set<int> out;
  for (int e : local)
    if (!unsafe.count(e) && g.nodes[e].numel() == R * C && g.nodes[e].dtype == SFX_F32) out.insert(e);
  return out;
}

// Row template with TMA bulk-copy staging: persistent warps, one row per warp
// per iteration; the row-local [R, C] inputs of the next NBUF rows are
// streamed into shared memory by cp.async.bulk (the TMA engine) and tracked by
// an mbarrier per stage, so HBM reads run continuously behind the arithmetic.
KernelSource lower_row_pipe(const Ctx& c, const RowPlan& rp, const std::set<int>& staged_inputs,
                            const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "row";
  ks.entry = "sfx_rowp_" + c.name;
  fill_common(c, ks);
  const int64_t R = rp.R, C = rp.C;
  const int V = 4, TPR = 32;
  const int64_t NCH = C / (TPR * V);
  const int WARPS = o.pipe_warps > 0 ? std::min(o.pipe_warps, 32) : 4;
  const int NBUF = o.pipe_stages > 0 ? std::min(o.pipe_stages, 8) : 2;
  std::vector<int> staged(staged_inputs.begin(), staged_inputs.end());
  const int64_t row_bytes = C * 4;
  const int64_t stage_bytes = row_bytes * static_cast<int64_t>(staged.size());
  const int64_t data_bytes = WARPS * NBUF * stage_bytes;
  const int smem = static_cast<int>(data_bytes + WARPS * NBUF * 8);
  if (smem > 227 * 1024) throw Error(SFX_ERR_UNSUPPORTED, "TMA row pipeline stages exceed shared memory");
  int ctas_per_sm = std::max(1, std::min<int>(8, static_cast<int>((220 * 1024) / smem)));
  if (o.pipe_ctas_per_sm > 0) ctas_per_sm = std::min(ctas_per_sm, o.pipe_ctas_per_sm);
  const int64_t grid = std::min<int64_t>((R + WARPS - 1) / WARPS, int64_t{kNumSMs} * ctas_per_sm);

  Emitter em(c.g, c.p, V, c.wide);
  em.rcp_reduced_divisors = rcp_divisors();
  std::string sig = signature(c, em, ks.entry, WARPS * 32);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  body.line("extern __shared__ __align__(128) unsigned char sfx_smem[];");
  body.line("const int lr = threadIdx.x & 31, warp = threadIdx.x >> 5;");
  body.line("const sfx_u32 gmask = 0xffffffffu;");
  body.line("const int gleader = 0;");
  body.line("unsigned long long* bars = (unsigned long long*)(sfx_smem + " + fmt_i(data_bytes) + ") + warp * " +
            std::to_string(NBUF) + ";");
  body.line("unsigned char* stages = sfx_smem + (" + it + ")warp * " + fmt_i(NBUF * stage_bytes) + ";");
  body.line("if (lr == 0) {");
  body.line("  for (int s = 0; s < " + std::to_string(NBUF) + "; ++s) sfx_mbar_init(bars + s, 1);");
  body.line("  sfx_fence_mbar_init();");
  body.line("}");
  body.line("__syncwarp();");
  body.line("const " + it + " row0 = (" + it + ")blockIdx.x * " + std::to_string(WARPS) + " + warp;");
  body.line("const " + it + " rstride = (" + it + ")gridDim.x * " + std::to_string(WARPS) + ";");
  // issue(stage, row): expect_tx + one bulk copy per staged input
  auto issue = [&](const std::string& s, const std::string& r) {
    body.line("{");
    body.line("  unsigned long long* bar = bars + " + s + ";");
    body.line("  sfx_mbar_expect_tx(bar, " + fmt_i(stage_bytes) + "u);");
    for (size_t k = 0; k < staged.size(); ++k)
      body.line("  sfx_bulk_g2s(stages + " + s + " * " + fmt_i(stage_bytes) + " + " +
                fmt_i(static_cast<int64_t>(k) * row_bytes) + ", " + em.input_ptr.at(staged[k]) + " + (" + r +
                ") * " + fmt_i(C) + ", " + fmt_i(row_bytes) + "u, bar);");
    body.line("}");
  };
  body.line("if (lr == 0) {");
  body.indent++;
  for (int s = 0; s < NBUF; ++s) {
    body.line("if (row0 + " + std::to_string(s) + " * rstride < " + fmt_i(R) + ")");
    issue(std::to_string(s), "row0 + " + std::to_string(s) + " * rstride");
  }
  body.indent--;
  body.line("}");
  body.line("for (int itr = 0;; ++itr) {");
  body.indent++;
  body.line("const " + it + " row = row0 + (" + it + ")itr * rstride;");
  body.line("if (row >= " + fmt_i(R) + ") break;");
  body.line("const int stg = itr % " + std::to_string(NBUF) + ";");
  body.line("sfx_mbar_wait(bars + stg, (unsigned)((itr / " + std::to_string(NBUF) + ") & 1));");
  em.push();
  std::string rbase = em.ivar(Emitter::imul("row", C));
  for (size_t k = 0; k < staged.size(); ++k) {
    std::string p = em.fresh("st");
    body.line("const float* " + p + " = (const float*)(stages + stg * " + fmt_i(stage_bytes) + " + " +
              fmt_i(static_cast<int64_t>(k) * row_bytes) + ");");
    em.staged[staged[k]] = {p, rbase};
  }
  emit_row_body(c, rp, em, body, TPR, V, NCH);
  em.pop();
  em.staged.clear();
  body.line("__syncwarp();");
  body.line("if (lr == 0 && row + " + std::to_string(NBUF) + " * rstride < " + fmt_i(R) + ")");
  issue("stg", "row + " + std::to_string(NBUF) + " * rstride");
  body.indent--;
  body.line("}");
  ks.code = assemble(sig, body);
  ks.block = WARPS * 32;
  ks.grid_x = grid;
  ks.smem = smem;
  ks.vector_width = V;
  ks.note = "rows=" + std::to_string(R) + " cols=" + std::to_string(C) + " TMA-staged inputs=" +
            std::to_string(staged.size()) + " stages=" + std::to_string(NBUF) + " persistent grid=" +
            std::to_string(grid) + " levels=" + std::to_string(rp.max_level);
  return ks;
}

// Resident rows (row_pipeline=4): for groups whose row-local inputs fit the
// shared memory of the whole GPU (148 x ~220 KB), one CTA per SM owns a
// contiguous, balanced range of rows (R/148 rounded either way) and its warps
// have the TMA engine copy EVERY one of those rows into shared memory at entry
// (one cp.async.bulk + mbarrier per row): the whole tensor is in flight at
// once, so the launch never runs a second wave or a partial last wave, and
// each warp starts a row as soon as that row has landed.  Rows are then
// processed like the register template (one warp per row, values from
// shared memory), roots stored straight from registers.
KernelSource lower_row_res(const Ctx& c, const RowPlan& rp, const std::set<int>& staged_inputs,
                           const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "row";
  ks.entry = "sfx_rowr_" + c.name;
  fill_common(c, ks);
  const int64_t R = rp.R, C = rp.C;
  const int V = 4, TPR = 32;
  const int64_t NCH = C / (TPR * V);
  std::vector<int> staged(staged_inputs.begin(), staged_inputs.end());
  const int64_t row_bytes = C * 4;
  const int64_t stage_bytes = row_bytes * static_cast<int64_t>(staged.size());
  const int64_t G = std::min<int64_t>(R, kNumSMs);
  const int64_t RPB = (R + G - 1) / G;  // most rows one CTA owns
  const int64_t data_bytes = RPB * stage_bytes;
  const int smem = static_cast<int>(data_bytes + RPB * 8);
  if (smem > 227 * 1024) throw Error(SFX_ERR_UNSUPPORTED, "resident rows exceed the shared memory of one CTA per SM");
  const int WARPS = static_cast<int>(std::min<int64_t>(RPB, o.pipe_warps > 0 ? std::min(o.pipe_warps, 32) : 32));

  Emitter em(c.g, c.p, V, c.wide);
  em.rcp_reduced_divisors = rcp_divisors();
  std::string sig = signature(c, em, ks.entry, WARPS * 32);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  body.line("extern __shared__ __align__(128) unsigned char sfx_smem[];");
  body.line("const int lr = threadIdx.x & 31, warp = threadIdx.x >> 5;");
  body.line("const sfx_u32 gmask = 0xffffffffu;");
  body.line("const int gleader = 0;");
  body.line("unsigned long long* bars = (unsigned long long*)(sfx_smem + " + fmt_i(data_bytes) + ");");
  // balanced contiguous ranges: CTA b owns rows [b*R/G, (b+1)*R/G)
  body.line("const " + it + " lo = (" + it + ")(((long long)blockIdx.x * " + fmt_i(R) + ") / " + fmt_i(G) + ");");
  body.line("const int nrows = (int)((((long long)blockIdx.x + 1) * " + fmt_i(R) + ") / " + fmt_i(G) + " - lo);");
  // every warp arms and issues its own rows (only that warp waits on them)
  body.line("if (lr == 0) {");
  body.line("  for (int j = warp; j < nrows; j += " + std::to_string(WARPS) + ") sfx_mbar_init(bars + j, 1);");
  body.line("  sfx_fence_mbar_init();");
  body.line("  for (int j = warp; j < nrows; j += " + std::to_string(WARPS) + ") {");
  body.line("    sfx_mbar_expect_tx(bars + j, " + fmt_i(stage_bytes) + "u);");
  for (size_t k = 0; k < staged.size(); ++k)
    body.line("    sfx_bulk_g2s(sfx_smem + (" + it + ")j * " + fmt_i(stage_bytes) + " + " +
              fmt_i(static_cast<int64_t>(k) * row_bytes) + ", " + em.input_ptr.at(staged[k]) + " + (lo + j) * " +
              fmt_i(C) + ", " + fmt_i(row_bytes) + "u, bars + j);");
  body.line("  }");
  body.line("}");
  body.line("__syncwarp();");
  body.line("for (int j = warp; j < nrows; j += " + std::to_string(WARPS) + ") {");
  body.indent++;
  body.line("const " + it + " row = lo + j;");
  body.line("sfx_mbar_wait(bars + j, 0u);");
  em.push();
  std::string rbase = em.ivar(Emitter::imul("row", C));
  for (size_t k = 0; k < staged.size(); ++k) {
    std::string p = em.fresh("st");
    body.line("const float* " + p + " = (const float*)(sfx_smem + (" + it + ")j * " + fmt_i(stage_bytes) + " + " +
              fmt_i(static_cast<int64_t>(k) * row_bytes) + ");");
    em.staged[staged[k]] = {p, rbase};
  }
  emit_row_body(c, rp, em, body, TPR, V, NCH);
  em.pop();
  em.staged.clear();
  body.indent--;
  body.line("}");
  ks.code = assemble(sig, body);
  ks.block = WARPS * 32;
  ks.grid_x = G;
  ks.smem = smem;
  ks.vector_width = V;
  ks.note = "rows=" + std::to_string(R) + " cols=" + std::to_string(C) + " resident rows: " + std::to_string(G) +
            " CTAs x " + std::to_string(WARPS) + " warps, <= " + std::to_string(RPB) +
            " rows per CTA copied into shared memory at entry (TMA), inputs=" + std::to_string(staged.size()) +
            " levels=" + std::to_string(rp.max_level);
  return ks;
}

}  // namespace lw
}  // namespace sfx
