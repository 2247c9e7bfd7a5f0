// Column-reduction templates: col (last-CTA combine, cross-rank) and colbc (grid barriers).
#include "lower_impl.hpp"

namespace sfx {
namespace lw {

// ---- COL ------------------------------------------------------------------------

// Components of a node of `dims` at position (o, r, i) of an [O | R | I]
// iteration space (o outer, r reduced, i inner), through a clean prefix split
// of the dims when there is one, else through the linear index (o*R + r)*I + i.
std::vector<Ix> orc_comps(Emitter& em, const std::vector<int64_t>& dims, int64_t O, int64_t R, int64_t I,
                          const Ix& o, const Ix& r, const Ix& i) {
  int k0 = prefix_split(dims, O);
  int k1 = k0 < 0 ? -1 : prefix_split(dims, O * R);
  if (k0 >= 0 && k1 >= k0 && prod(dims, k1, dims.size()) == I && prod(dims, k0, k1) == R) {
    std::vector<int64_t> d0(dims.begin(), dims.begin() + k0), d1(dims.begin() + k0, dims.begin() + k1),
        d2(dims.begin() + k1, dims.end());
    std::vector<Ix> a = em.from_linear(o, d0), b = em.from_linear(r, d1), c = em.from_linear(i, d2);
    a.insert(a.end(), b.begin(), b.end());
    a.insert(a.end(), c.begin(), c.end());
    return a;
  }
  std::string ob = em.ivar(Emitter::imul(em.ivar(Emitter::iadd(Emitter::imul(o.e, R), r.e)), I));
  Ix L;
  if (i.kind == IX_PLUS) {
    L = em.lane_plus(em.ivar(Emitter::iadd(ob, i.base)));
  } else {
    L = em.uni(em.ivar(Emitter::iadd(ob, i.e)));
    L.kind = i.kind;
  }
  return em.from_linear(L, dims);
}

// Column template generalised to [outer | reduced | inner]: the reduce
// operand's reduced dims are contiguous; "columns" are the O x I kept elements
// (C3: O = 1).  A warp covers CL column vectors x RL rows (RL > 1 when there are
// fewer than 32 column vectors, e.g. full reductions), 8 warps stride the rows
// of a stripe, stripes combine in a single launch (last-CTA ticket).
KernelSource lower_col(const Ctx& c, const ColPlan& cp, const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "col";
  ks.entry = "sfx_col_" + c.name;
  fill_common(c, ks);
  const int64_t O = cp.O, R = cp.R, I = cp.I, C = cp.O * cp.I;
  const int V = (I % 4 == 0) ? 4 : 1;
  const int64_t cvec = (C + V - 1) / V;
  int CL = 1;
  while (CL < 32 && CL < cvec) CL *= 2;
  const int RL = 32 / CL;
  const int WARPS = 8, B = WARPS * 32;
  const int RSUB = WARPS * RL;  // row sub-streams per CTA
  const int64_t TC = static_cast<int64_t>(CL) * V;
  const int64_t tiles = (C + TC - 1) / TC;
  // row stripes: 2 CTAs per SM in exactly one wave, each thread keeping 16
  // rows x (streamed inputs) 128-bit loads in flight under a 128-register cap
  // (__launch_bounds__(256, 2)).  Measured on C3 (tools/gpu_ab_col.sh): 4 CTAs/SM
  // x 4 rows 94.5 us, 4 x 8 rows 88.5 us, 2 x 16 rows 84.3 us (0.99 of the
  // measured copy peak; a torch read-only sum of the same bytes takes 94.6 us).
  // The col template reuses rows_per_cta as a stripe-count override,
  // items_per_thread as rows per iteration and pipe_ctas_per_sm as the
  // residency target.
  const int ctas_per_sm = o.pipe_ctas_per_sm > 0 ? o.pipe_ctas_per_sm : 2;
  int64_t S = o.rows_per_cta > 0 ? o.rows_per_cta : std::max<int64_t>(1, kNumSMs * ctas_per_sm / tiles);
  S = std::min<int64_t>(S, std::max<int64_t>(1, R / (8 * RSUB)));
  S = std::min<int64_t>(S, 65535);
  const int64_t RS = (R + S - 1) / S;
  const int NR = static_cast<int>(c.reduces.size());

  Emitter em(c.g, c.p, V, c.wide);
  em.rcp_reduced_divisors = rcp_divisors();
  std::string sig = signature(c, em, ks.entry, B, ctas_per_sm);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  // workspace: tickets[tiles] (256-B padded), then partials[NR][S][C]
  const int64_t ticket_words = (tiles + 63) / 64 * 64;
  // float sums accumulate in double end to end (per-thread, CTA and stripe
  // combines): a column of 65,536 fp32 terms with cancellation is otherwise
  // off by ~eps*sum|x| (SURVEY §7 hard part 1); max/min/i32 are exact anyway.
  auto acc_t = [&](int k) -> std::string {
    const Node& rn = c.g.nodes[c.reduces[k]];
    return (rn.reducer == SFX_REDUCE_SUM && rn.dtype == SFX_F32) ? "double" : ctype(rn.dtype);
  };
  auto fold_fn = [&](int k) -> const char* {
    const Node& rn = c.g.nodes[c.reduces[k]];
    return rn.reducer == SFX_REDUCE_SUM ? "sfx_fold_sum" : rn.reducer == SFX_REDUCE_MAX ? "sfx_fold_pmax"
                                                                                          : "sfx_fold_pmin";
  };
  std::vector<int64_t> part_word(NR);
  int64_t words = ticket_words;
  for (int k = 0; k < NR; ++k) {
    part_word[k] = words;
    words += S * C * (acc_t(k) == "double" ? 2 : 1);
    words = (words + 63) / 64 * 64;
  }
  const int64_t seq_word = words;
  if (c.peer) {
    words += (tiles + 63) / 64 * 64;
    ks.peer_bytes = ((2LL * SFX_PEER_MAX_RANKS * NR * C + 2LL * NR * C) * 8 + tiles * SFX_PEER_MAX_RANKS * 4 + 255) /
                    256 * 256;
  }
  ks.workspace_bytes = words * 4;

  body.line("const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;");
  body.line("const int cl = lane & " + std::to_string(CL - 1) + ", rl = lane / " + std::to_string(CL) + ";");
  body.line("const int rsub = warp * " + std::to_string(RL) + " + rl;");
  body.line("const " + it + " c0 = (" + it + ")blockIdx.x * " + fmt_i(TC) + " + cl * " + std::to_string(V) + ";");
  body.line("const bool cok = c0 < " + fmt_i(C) + ";");
  body.line("const " + it + " r_begin = (" + it + ")blockIdx.y * " + fmt_i(RS) + ";");
  body.line("const " + it + " r_end = min((" + it + ")" + fmt_i(R) + ", r_begin + " + fmt_i(RS) + ");");
  // the column vector's outer / inner coordinates (a vector never crosses an
  // outer index: I % V == 0)
  body.line("const " + it + " co = c0 / " + fmt_i(I) + ", ci = c0 % " + fmt_i(I) + ";");
  std::vector<std::vector<std::string>> acc(NR, std::vector<std::string>(V));
  for (int k = 0; k < NR; ++k) {
    const Node& rn = c.g.nodes[c.reduces[k]];
    std::string init;
    if (rn.reducer == SFX_REDUCE_SUM) init = rn.dtype == SFX_F32 ? "0.0" : "0";
    else if (rn.dtype == SFX_F32) init = "sfx_bits_f(0x7fc00000)";  // NaN = identity of fmaxf/fminf
    else init = rn.reducer == SFX_REDUCE_MAX ? "(int)0x80000000u" : "0x7fffffff";
    for (int l = 0; l < V; ++l) {
      acc[k][l] = em.fresh("acc");
      body.line(acc_t(k) + " " + acc[k][l] + " = " + init + ";");
    }
  }
  std::vector<int> full_roots, col_roots;
  for (int r : c.p.roots) (c.dep.at(r) || c.g.nodes[r].numel() != R * C ? col_roots : full_roots).push_back(r);
  auto inner_ix = [&](int lane) {
    em.lane = lane;
    return V == 1 ? em.uni("ci") : em.lane_plus("ci");
  };

  // one row of this thread's column vector: elementwise roots stored, reduce
  // operands folded into the per-lane accumulators
  auto emit_row = [&](const std::string& r) {
    Ix rix = em.uni(r), oix = em.uni("co");
    std::vector<std::vector<std::string>> fv(full_roots.size(), std::vector<std::string>(V));
    std::vector<std::vector<std::string>> faddr(full_roots.size(), std::vector<std::string>(V));
    std::vector<bool> fvec(full_roots.size(), V == 4);
    for (int lane = 0; lane < V; ++lane) {
      Ix iix = inner_ix(lane);
      for (size_t k = 0; k < full_roots.size(); ++k) {
        std::vector<Ix> comps = orc_comps(em, c.g.nodes[full_roots[k]].dims, O, R, I, oix, rix, iix);
        fv[k][lane] = em.value(full_roots[k], comps);
        Ix L = em.linearize(comps, c.g.nodes[full_roots[k]].dims);
        faddr[k][lane] = lane == 0 && L.kind == IX_PLUS ? L.base : L.e;
        if (lane == 0 && L.kind != IX_PLUS) fvec[k] = false;
      }
      for (int k = 0; k < NR; ++k) {
        const Node& rn = c.g.nodes[c.reduces[k]];
        const Node& in = c.g.nodes[rn.operands[0]];
        std::string v = em.value(rn.operands[0], orc_comps(em, in.dims, O, R, I, oix, rix, iix));
        body.line(acc[k][lane] + " = " + fold_fn(k) + "(" + acc[k][lane] + ", " + v + ");");
      }
    }
    for (size_t k = 0; k < full_roots.size(); ++k) {
      std::string out = "out" + std::to_string(root_slot(c, full_roots[k]));
      if (fvec[k])
        body.line("sfx_st4(" + out + " + " + faddr[k][0] + ", " + fv[k][0] + ", " + fv[k][1] + ", " + fv[k][2] +
                  ", " + fv[k][3] + ");");
      else
        for (int l = 0; l < V; ++l) body.line(out + "[" + faddr[k][l] + "] = " + fv[k][l] + ";");
    }
  };
  // UR rows per iteration, unguarded, so all their 128-bit loads are in flight
  // together; then the remainder one row at a time
  const int UR = o.items_per_thread > 0 ? std::min(o.items_per_thread, 32) : 16;
  body.line("if (cok) {");
  body.indent++;
  body.line(it + " r = r_begin + rsub;");
  body.line("for (; r + " + std::to_string((UR - 1) * RSUB) + " < r_end; r += " + std::to_string(UR * RSUB) + ") {");
  body.indent++;
  em.push();
  for (int u = 0; u < UR; ++u) {
    std::string ru = "r" + std::to_string(u);
    body.line("const " + it + " " + ru + " = r + " + std::to_string(u * RSUB) + ";");
    emit_row(ru);
  }
  em.pop();
  body.indent--;
  body.line("}");
  body.line("for (; r < r_end; r += " + std::to_string(RSUB) + ") {");
  body.indent++;
  em.push();
  emit_row("r");
  em.pop();
  body.indent--;
  body.line("}");
  body.indent--;
  body.line("}");

  // CTA combine through shared memory (deterministic row-substream order)
  for (int k = 0; k < NR; ++k) {
    const std::string T = acc_t(k);
    body.line("__shared__ " + T + " sp" + std::to_string(k) + "[" + std::to_string(RSUB) + "][" + fmt_i(TC) + "];");
    for (int l = 0; l < V; ++l)
      body.line("sp" + std::to_string(k) + "[rsub][cl * " + std::to_string(V) + " + " + std::to_string(l) +
                "] = " + acc[k][l] + ";");
  }
  body.line("__syncthreads();");
  body.line("unsigned* tickets = ws;");
  body.line("const bool lead = warp == 0 && rl == 0 && cok;");
  body.line("if (lead) {");
  body.indent++;
  for (int k = 0; k < NR; ++k) {
    const std::string T = acc_t(k);
    std::string part = "part" + std::to_string(k);
    body.line(T + "* " + part + " = (" + T + "*)(ws + " + fmt_i(part_word[k]) + ");");
    for (int l = 0; l < V; ++l) {
      std::string sidx = "cl * " + std::to_string(V) + " + " + std::to_string(l);
      std::string t = em.fresh("t");
      body.line(T + " " + t + " = sp" + std::to_string(k) + "[0][" + sidx + "];");
      body.line("for (int w = 1; w < " + std::to_string(RSUB) + "; ++w) " + t + " = " + fold_fn(k) + "(" + t +
                ", sp" + std::to_string(k) + "[w][" + sidx + "]);");
      body.line(part + "[(" + it + ")blockIdx.y * " + fmt_i(C) + " + c0 + " + std::to_string(l) + "] = " + t + ";");
    }
  }
  body.indent--;
  body.line("}");
  body.line("__threadfence();");
  body.line("__syncthreads();");
  body.line("__shared__ unsigned s_last;");
  body.line("if (threadIdx.x == 0) s_last = (atomicAdd(&tickets[blockIdx.x], 1u) == gridDim.y - 1u);");
  body.line("__syncthreads();");
  body.line("if (!s_last) return;");
  body.line("__threadfence();");
  // finisher: ordered combine over stripes (then, with cross_rank, over ranks
  // in rank order through peer memory), then the column roots
  const std::string Cs = fmt_i(C);
  auto stripe_total = [&](int k) {
    const std::string T = acc_t(k);
    std::string part = "fp" + std::to_string(k);
    body.line("const " + T + "* " + part + " = (const " + T + "*)(ws + " + fmt_i(part_word[k]) + ") + c0;");
    std::vector<std::string> tv(V);
    for (int l = 0; l < V; ++l) {
      tv[l] = em.fresh("tot");
      body.line(T + " " + tv[l] + " = __ldcg(" + part + " + " + std::to_string(l) + ");");
    }
    body.line("for (" + it + " s = 1; s < " + fmt_i(S) + "; ++s) {");
    for (int l = 0; l < V; ++l)
      body.line("  " + tv[l] + " = " + fold_fn(k) + "(" + tv[l] + ", __ldcg(" + part + " + s * " + Cs + " + " +
                std::to_string(l) + "));");
    body.line("}");
    return tv;
  };
  // the sequential fold's first element (row 0 of the column; with
  // cross_rank, row 0 of rank 0's shard)
  auto first_elem = [&](int k, int l) {
    const Node& rn = c.g.nodes[c.reduces[k]];
    const Node& in = c.g.nodes[rn.operands[0]];
    Ix iix = inner_ix(l);
    return em.value(rn.operands[0], orc_comps(em, in.dims, O, R, I, em.uni("co"), em.uni("0"), iix));
  };
  auto needs_first = [&](int k) {
    const Node& rn = c.g.nodes[c.reduces[k]];
    return rn.reducer != SFX_REDUCE_SUM && rn.dtype == SFX_F32;
  };
  std::map<int, std::vector<std::string>> total;
  // peer arena layout (8-byte slots): data[2][PMAX][NR][C], first[2][NR][C],
  // then flags[tiles][PMAX] (u32); local ws keeps one sequence word per tile
  const int PMAX = SFX_PEER_MAX_RANKS;
  const int64_t first_slot = 2LL * PMAX * NR * C;
  const int64_t flag_byte = (first_slot + 2LL * NR * C) * 8;
  // per reduce and lane: the column total in the accumulation type, declared
  // at CTA scope so the cross-rank protocol can sit between its two halves
  std::vector<std::vector<std::string>> ptot(NR, std::vector<std::string>(V));
  if (c.peer) {
    for (int k = 0; k < NR; ++k)
      for (int l = 0; l < V; ++l) {
        ptot[k][l] = em.fresh("ptot");
        body.line(acc_t(k) + " " + ptot[k][l] + " = 0;");
      }
    body.line("__shared__ unsigned s_seq;");
    body.line("if (threadIdx.x == 0) { const unsigned q = ws[" + fmt_i(seq_word) +
              " + blockIdx.x] + 1u; ws[" + fmt_i(seq_word) + " + blockIdx.x] = q; s_seq = q; }");
    body.line("__syncthreads();");
    body.line("const unsigned seq = s_seq;");
    body.line("const long long par = seq & 1u;");
    body.line("if (lead) {");
    body.indent++;
    em.push();
    for (int k = 0; k < NR; ++k) {
      const std::string T = acc_t(k);
      std::vector<std::string> tv = stripe_total(k);
      for (int l = 0; l < V; ++l) body.line(ptot[k][l] + " = " + tv[l] + ";");
      // a single rank has nothing to exchange: the protocol only runs for pn > 1
      body.line("for (int p = 0; p < pn && pn > 1; ++p) {");
      body.line("  unsigned long long* slot = (unsigned long long*)(peers[p] + poff) + ((par * " +
                std::to_string(PMAX) + " + prank) * " + std::to_string(NR) + " + " + std::to_string(k) + ") * " + Cs +
                " + c0;");
      for (int l = 0; l < V; ++l) body.line("  *(" + T + "*)(slot + " + std::to_string(l) + ") = " + tv[l] + ";");
      if (needs_first(k)) {
        body.line("  if (prank == 0) {");
        body.line("    float* f = (float*)((unsigned long long*)(peers[p] + poff) + " + fmt_i(first_slot) +
                  " + (par * " + std::to_string(NR) + " + " + std::to_string(k) + ") * " + Cs + " + c0);");
        for (int l = 0; l < V; ++l) body.line("    f[" + std::to_string(2 * l) + "] = " + first_elem(k, l) + ";");
        body.line("  }");
      }
      body.line("}");
    }
    em.pop();
    body.indent--;
    body.line("}");
    // the lead lanes' stores reach thread p through the CTA barrier; its
    // release store at system scope is cumulative over them (no separate
    // __threadfence_system: it cost 2 us on the critical path)
    body.line("if (pn > 1) {");
    body.line("  __syncthreads();");
    body.line("  if (threadIdx.x < pn) {");
    body.line("    sfx_st_release_sys((unsigned*)(peers[threadIdx.x] + poff + " + fmt_i(flag_byte) +
              ") + blockIdx.x * " + std::to_string(PMAX) + " + prank, seq);");
    body.line("    sfx_peer_wait((const unsigned*)(peers[prank] + poff + " + fmt_i(flag_byte) + ") + blockIdx.x * " +
              std::to_string(PMAX) + " + threadIdx.x, seq);");
    body.line("  }");
    body.line("  __syncthreads();");
    body.line("}");
  }
  body.line("if (lead) {");
  body.indent++;
  em.push();
  for (int k = 0; k < NR; ++k) {
    const Node& rn = c.g.nodes[c.reduces[k]];
    const std::string T = acc_t(k);
    std::vector<std::string> tv;
    std::string first_peer;  // pn > 1: rank 0's published first element (per lane, below)
    if (c.peer) {
      // every rank folds the same slots in rank order: bit-identical results
      body.line("if (pn > 1) {");
      body.line("  const unsigned long long* xs = (const unsigned long long*)(peers[prank] + poff) + (par * " +
                std::to_string(PMAX) + " * " + std::to_string(NR) + " + " + std::to_string(k) + ") * " + Cs + " + c0;");
      for (int l = 0; l < V; ++l)
        body.line("  " + ptot[k][l] + " = __ldcv((const " + T + "*)(xs + " + std::to_string(l) + "));");
      body.line("  for (int q = 1; q < pn; ++q) {");
      for (int l = 0; l < V; ++l)
        body.line("    " + ptot[k][l] + " = " + fold_fn(k) + "(" + ptot[k][l] + ", __ldcv((const " + T +
                  "*)(xs + (long long)q * " + std::to_string(NR) + " * " + Cs + " + " + std::to_string(l) + ")));");
      body.line("  }");
      body.line("}");
      tv = ptot[k];
    } else {
      tv = stripe_total(k);
    }
    if (T == "double")
      for (int l = 0; l < V; ++l) {
        std::string fv32 = em.fresh("tot");
        body.line("const float " + fv32 + " = (float)" + tv[l] + ";");
        tv[l] = fv32;
      }
    if (needs_first(k)) {
      // sequential std::max/min fold semantics: a NaN first element wins
      for (int l = 0; l < V; ++l) {
        std::string f0 = first_elem(k, l);
        if (c.peer) {
          std::string fp = em.fresh("f0");
          body.line("const float " + fp + " = pn > 1 ? __ldcv((const float*)((const unsigned long long*)(peers[prank] + poff) + " +
                    fmt_i(first_slot) + " + (par * " + std::to_string(NR) + " + " + std::to_string(k) + ") * " + Cs +
                    " + c0 + " + std::to_string(l) + ")) : " + f0 + ";");
          f0 = fp;
        }
        body.line(tv[l] + " = sfx_fold_first(" + f0 + ", " + tv[l] + ");");
      }
    }
    (void)rn;
    total[c.reduces[k]] = tv;
  }
  em.resolve = [&](int node, const std::vector<Ix>&) -> std::string {
    auto f = total.find(node);
    if (f == total.end()) return "";
    return f->second[em.lane];
  };
  for (int r : col_roots) {
    std::vector<std::string> v(V);
    for (int l = 0; l < V; ++l) {
      em.lane = l;
      Ix col = V == 1 ? em.uni("c0") : em.lane_plus("c0");
      v[l] = em.value(r, em.from_linear(col, c.g.nodes[r].dims));
    }
    std::string out = "out" + std::to_string(root_slot(c, r));
    if (V == 4)
      body.line("sfx_st4(" + out + " + c0, " + v[0] + ", " + v[1] + ", " + v[2] + ", " + v[3] + ");");
    else
      body.line(out + "[c0] = " + v[0] + ";");
  }
  em.pop();
  body.indent--;
  body.line("}");
  body.line("if (threadIdx.x == 0) tickets[blockIdx.x] = 0u;");
  ks.code = assemble(sig, body);
  ks.block = B;
  ks.grid_x = tiles;
  ks.grid_y = S;
  ks.vector_width = V;
  ks.note = "outer=" + std::to_string(O) + " reduced=" + std::to_string(R) + " inner=" + std::to_string(I) +
            " tiles=" + std::to_string(tiles) + " stripes=" + std::to_string(S) + " lanes(col x row)=" +
            std::to_string(CL) + "x" + std::to_string(RL);
  return ks;
}

// Second moments folded in the first-level pass (lower_impl.hpp).
std::vector<Var2> find_var2(const Ctx& c, const std::map<int, int>& level, int max_level) {
  const Graph& g = c.g;
  std::vector<Var2> out;
  if (max_level != 2 || c.peer) return out;
  const char* env = std::getenv("SFX_COLBC_TWO_PASS");
  if (env && env[0] == '1') return out;
  auto is_ew = [&](int n, int kind) { return g.nodes[n].op == SFX_OP_ELEMENTWISE && g.nodes[n].kind == kind; };
  auto sum_f32 = [&](int n) {
    const Node& x = g.nodes[n];
    return x.op == SFX_OP_REDUCE && x.reducer == SFX_REDUCE_SUM && x.dtype == SFX_F32;
  };
  for (int b : c.reduces) {
    if (level.at(b) != 2) continue;
    if (!sum_f32(b)) return {};
    const int sq = g.nodes[b].operands[0];
    if (!c.p.is_member(sq) || !is_ew(sq, SFX_EW_MUL) || g.nodes[sq].operands[0] != g.nodes[sq].operands[1]) return {};
    const int d = g.nodes[sq].operands[0];
    if (!c.p.is_member(d) || !is_ew(d, SFX_EW_SUB)) return {};
    bool found = false;
    for (int side = 0; side < 2 && !found; ++side) {
      const int u = g.nodes[d].operands[side], mb = g.nodes[d].operands[1 - side];
      if (!c.p.is_member(mb) || g.nodes[mb].op != SFX_OP_BROADCAST) continue;
      int m = g.nodes[mb].operands[0];
      int a = m;
      if (c.p.is_member(m) && is_ew(m, SFX_EW_SCALE)) a = g.nodes[m].operands[0];
      if (!c.p.is_member(a) || !sum_f32(a) || level.count(a) == 0 || level.at(a) != 1) continue;
      const Node& an = g.nodes[a];
      if (an.operands[0] != u || an.reduce_dims != g.nodes[b].reduce_dims) continue;
      if (g.nodes[mb].dims != g.nodes[u].dims || g.nodes[u].dtype != SFX_F32) continue;
      std::vector<int64_t> kept;
      for (int64_t k = 0; k < g.nodes[u].rank(); ++k)
        if (std::find(an.reduce_dims.begin(), an.reduce_dims.end(), k) == an.reduce_dims.end()) kept.push_back(k);
      if (g.nodes[mb].dim_map != kept) continue;
      out.push_back({a, b, u, mb});
      found = true;
    }
    if (!found) return {};
  }
  return out;
}

// Column reductions broadcast back (batch-norm): one launch, a co-resident
// grid of column tiles x row stripes (2 CTAs/SM, one wave, cooperative
// launch).  Per reduction level: every CTA folds its stripe (per-lane fp64
// accumulators for f32 sums), combines its warps through shared memory and
// writes a partial; a grid barrier; then every thread folds the S stripe
// partials of its own columns in stripe order (identical totals in every CTA)
// and keeps them in registers, where the broadcast-back reads them.  A final
// pass writes the element roots.  Passes after the first re-read the stripe,
// mostly from L2 (batch-norm [65536, 256]: 64 MB).
KernelSource lower_colbc(const Ctx& c, const ColBcPlan& bp, const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "colbc";
  ks.entry = "sfx_colbc_" + c.name;
  fill_common(c, ks);
  const int64_t O = bp.O, R = bp.R, I = bp.I, C = O * I;
  const int V = (I % 4 == 0) ? 4 : 1;
  const int64_t cvec = (C + V - 1) / V;
  int CL = 1;
  while (CL < 32 && CL < cvec) CL *= 2;
  const int RL = 32 / CL;
  const int WARPS = 8, B = WARPS * 32;
  const int RSUB = WARPS * RL;
  const int64_t TC = static_cast<int64_t>(CL) * V;
  const int64_t tiles = (C + TC - 1) / TC;
  const int ctas_per_sm = o.pipe_ctas_per_sm > 0 ? std::min(o.pipe_ctas_per_sm, 8) : 2;
  if (tiles > int64_t{kNumSMs} * ctas_per_sm)
    throw Error(SFX_ERR_UNSUPPORTED, "colbc: " + std::to_string(tiles) + " column tiles exceed one co-resident wave");
  int64_t S = o.rows_per_cta > 0 ? o.rows_per_cta : std::max<int64_t>(1, kNumSMs * ctas_per_sm / tiles);
  S = std::min<int64_t>(S, std::max<int64_t>(1, R / RSUB));
  S = std::max<int64_t>(1, std::min<int64_t>(S, kNumSMs * ctas_per_sm / tiles));
  const int64_t RS = (R + S - 1) / S;
  int UR = o.items_per_thread > 0 ? std::min(o.items_per_thread, 16) : 8;
  const int NR = static_cast<int>(c.reduces.size());
  Emitter em(c.g, c.p, V, c.wide);
  em.rcp_reduced_divisors = rcp_divisors();
  std::string sig = signature(c, em, ks.entry, B, ctas_per_sm);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  auto acc_t = [&](int r) -> std::string {
    const Node& rn = c.g.nodes[r];
    return (rn.reducer == SFX_REDUCE_SUM && rn.dtype == SFX_F32) ? "double" : ctype(rn.dtype);
  };
  auto fold_fn = [&](int r) -> const char* {
    const Node& rn = c.g.nodes[r];
    return rn.reducer == SFX_REDUCE_SUM ? "sfx_fold_sum" : rn.reducer == SFX_REDUCE_MAX ? "sfx_fold_pmax"
                                                                                         : "sfx_fold_pmin";
  };
  // workspace: barrier counters (64 words), then per reduce partials[S][C] and totals[C] (8-byte slots)
  std::map<int, int64_t> part_word, tot_word;
  int64_t words = 64;  // [0] arrivals, [1] exits, [2] launch sequence (cross-rank)
  for (int r : c.reduces) {
    part_word[r] = words;
    words += S * C * 2;
    tot_word[r] = words;
    words += C * 2 + 64;
  }
  ks.workspace_bytes = words * 4;
  ks.cooperative = true;
  // cross-rank (SyncBatchNorm): per level, each rank's column totals are pushed
  // to every rank's peer arena (slots [2][PMAX][NR][C], 8 B) by the tile's first
  // stripe CTA, flagged per tile with the step number, and folded in rank order
  // by every thread.  Steps number (launch, level) pairs: launch_seq * L + lv.
  const int PMAX = SFX_PEER_MAX_RANKS;
  std::map<int, int> red_index;
  for (int k = 0; k < NR; ++k) red_index[c.reduces[k]] = k;
  const int64_t pflag_byte = (2LL * PMAX * NR * C) * 8;
  if (c.peer) {
    for (int r : c.reduces) {
      const Node& rn = c.g.nodes[r];
      if (rn.reducer != SFX_REDUCE_SUM && rn.dtype == SFX_F32)
        throw Error(SFX_ERR_UNSUPPORTED, "cross-rank colbc supports sum reductions (max/min NaN-first rule: col template)");
    }
    ks.peer_bytes = (pflag_byte + tiles * PMAX * 4 + 255) / 256 * 256;
  }
  body.line("const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;");
  body.line("const int cl = lane & " + std::to_string(CL - 1) + ", rl = lane / " + std::to_string(CL) + ";");
  body.line("const int rsub = warp * " + std::to_string(RL) + " + rl;");
  body.line("const " + it + " c0 = (" + it + ")blockIdx.x * " + fmt_i(TC) + " + cl * " + std::to_string(V) + ";");
  body.line("const bool cok = c0 < " + fmt_i(C) + ";");
  body.line("const " + it + " r_begin = (" + it + ")blockIdx.y * " + fmt_i(RS) + ";");
  body.line("const " + it + " r_end = min((" + it + ")" + fmt_i(R) + ", r_begin + " + fmt_i(RS) + ");");
  body.line("const " + it + " co = cok ? c0 / " + fmt_i(I) + " : 0, ci = cok ? c0 % " + fmt_i(I) + " : 0;");
  if (c.peer) body.line("const unsigned launch_seq = __ldcg(ws + 2);");
  auto inner_ix = [&](int lane) {
    em.lane = lane;
    return V == 1 ? em.uni("ci") : em.lane_plus("ci");
  };
  // totals of every finished level, per lane, in registers
  std::map<int, std::vector<std::string>> total;
  em.resolve = [&](int node, const std::vector<Ix>&) -> std::string {
    auto f = total.find(node);
    if (f == total.end()) {
      if (c.g.nodes[node].op == SFX_OP_REDUCE && !degenerate_reduce(c.g, c.g.nodes[node]))
        throw Error(SFX_ERR_INVALID, "internal: reduction used before it is combined");
      return "";
    }
    return f->second[em.lane];
  };
  // a pass over this CTA's stripe: UR rows per iteration (unguarded, loads in
  // flight together), then the remainder.  Passes alternate direction: every
  // CTA ends a pass on the rows it read last, which are the ones still in L2
  // when the grid starts the next pass, so a stripe set larger than L2 re-reads
  // its most recent rows from L2 instead of HBM (the fold order is the mirror
  // image: deterministic, a reduction-order difference).  SFX_COLBC_FORWARD=1:
  // every pass forward (A/B).
  // Staged inputs (the [O, R, I] inputs read only at the thread's own element):
  // a per-thread cp.async ring in dynamic shared memory keeps NS x UR rows of
  // them in flight per thread without holding them in registers (the register
  // passes are HBM/L2-latency bound at 2 CTAs/SM).  row_pipeline=1: register
  // passes (A/B).
  std::vector<int> stage_in;
  int NS = 0;
  if (V == 4 && o.row_pipeline != 1) {
    for (int e : identity_inputs(c, O * R * I)) stage_in.push_back(e);
    if (!stage_in.empty()) {
      // static shared memory: per reduce [RSUB][TC] partials + small arrays
      // (the CTA combine's partials live in the ring once a pass is done)
      const int64_t part = static_cast<int64_t>(NR) * RSUB * TC * 8;
      const int64_t budget = std::min<int64_t>(96 * 1024, (220 * 1024) / ctas_per_sm - 4096 - 1024);
      int64_t stage_bytes = static_cast<int64_t>(UR) * stage_in.size() * B * 16;
      NS = static_cast<int>(std::min<int64_t>(4, budget / stage_bytes));
      // several staged inputs: fewer rows per stage, same rows in flight
      while (NS < 2 && UR > 2 && o.items_per_thread == 0) {
        UR /= 2;
        stage_bytes /= 2;
        NS = static_cast<int>(std::min<int64_t>(4, budget / stage_bytes));
      }
      if (NS < 2 || NS * stage_bytes < part) {
        NS = 0;
        stage_in.clear();
      } else {
        ks.smem = static_cast<int>(NS * stage_bytes);
      }
    }
  }
  if (NS > 0) body.line("extern __shared__ __align__(128) unsigned char sfx_smem[];");
  const char* fwenv = std::getenv("SFX_COLBC_FORWARD");
  const bool alternate = !(fwenv && fwenv[0] == '1');
  int pass_no = 0;
  auto stripe_pass = [&](const std::function<void(const std::string&)>& row_fwd) {
    const bool rev = alternate && (pass_no++ % 2 == 1);
    auto row = [&](const std::string& rf) {
      if (!rev) return row_fwd(rf);
      const std::string rr = em.fresh("rr");
      body.line("const " + it + " " + rr + " = r_begin + r_end - 1 - (" + rf + ");");
      row_fwd(rr);
    };
    body.line("if (cok) {");
    body.indent++;
    const std::string r = em.fresh("r");
    body.line(it + " " + r + " = r_begin + rsub;");
    if (NS > 0) {
      // cp.async ring: chunk j = this thread's UR rows r_begin + rsub + (j*UR + u)*RSUB;
      // chunks j+1 .. j+NS-1 are in flight while chunk j is folded
      const std::string nch = em.fresh("nch"), j = em.fresh("j");
      body.line("const " + it + " " + nch + "_span = r_end - " + r + " - " + std::to_string((UR - 1) * RSUB) + ";");
      body.line("const int " + nch + " = " + nch + "_span > 0 ? (int)((" + nch + "_span + " +
                std::to_string(UR * RSUB - 1) + ") / " + std::to_string(UR * RSUB) + ") : 0;");
      // linear index (lane 0) of staged input k at stripe row `rr` and this thread's column
      auto base_of = [&](int k, const std::string& rr) {
        const Node& in = c.g.nodes[stage_in[k]];
        em.lane = 0;
        Ix L = em.linearize(orc_comps(em, in.dims, O, R, I, em.uni("co"), em.uni(rr), inner_ix(0)), in.dims);
        if (L.kind != IX_PLUS) throw Error(SFX_ERR_INVALID, "internal: colbc staged input is not vectorised");
        return L.base;
      };
      auto slot_ptr = [&](const std::string& slot, int u, int k) {
        return "(sfx_smem + ((((" + slot + ") * " + std::to_string(UR) + " + " + std::to_string(u) + ") * " +
               std::to_string(stage_in.size()) + " + " + std::to_string(k) + ") * " + std::to_string(B) +
               " + threadIdx.x) * 16)";
      };
      auto issue = [&](const std::string& jn) {
        em.push();
        for (int u = 0; u < UR; ++u) {
          std::string rf = em.fresh("rf");
          body.line("const " + it + " " + rf + " = " + r + " + ((" + it + ")(" + jn + ") * " + std::to_string(UR) + " + " +
                    std::to_string(u) + ") * " + std::to_string(RSUB) + ";");
          std::string rr = rf;
          if (rev) {
            rr = em.fresh("rr");
            body.line("const " + it + " " + rr + " = r_begin + r_end - 1 - (" + rf + ");");
          }
          for (size_t k = 0; k < stage_in.size(); ++k)
            body.line("sfx_cp_async16(" + slot_ptr("(" + jn + ") % " + std::to_string(NS), u, static_cast<int>(k)) +
                      ", " + em.input_ptr.at(stage_in[k]) + " + " + base_of(static_cast<int>(k), rr) + ");");
        }
        em.pop();
      };
      for (int k = 0; k < NS - 1; ++k) {
        body.line("if (" + std::to_string(k) + " < " + nch + ") {");
        body.indent++;
        issue(std::to_string(k));
        body.indent--;
        body.line("}");
        body.line("sfx_cp_async_commit();");
      }
      body.line("for (int " + j + " = 0; " + j + " < " + nch + "; ++" + j + ") {");
      body.indent++;
      body.line("if (" + j + " + " + std::to_string(NS - 1) + " < " + nch + ") {");
      body.indent++;
      issue(j + " + " + std::to_string(NS - 1));
      body.indent--;
      body.line("}");
      body.line("sfx_cp_async_commit();");
      body.line("sfx_cp_async_wait<" + std::to_string(NS - 1) + ">();  // chunk " + j + " landed (own copies only)");
      em.push();
      for (int u = 0; u < UR; ++u) {
        std::string rf = em.fresh("ru");
        body.line("const " + it + " " + rf + " = " + r + " + ((" + it + ")" + j + " * " + std::to_string(UR) + " + " +
                  std::to_string(u) + ") * " + std::to_string(RSUB) + ";");
        std::string rr = rf;
        if (rev) {
          rr = em.fresh("rr");
          body.line("const " + it + " " + rr + " = r_begin + r_end - 1 - (" + rf + ");");
        }
        for (size_t k = 0; k < stage_in.size(); ++k) {
          std::string sp = em.fresh("sp");
          body.line("const float* " + sp + " = (const float*)" + slot_ptr(j + " % " + std::to_string(NS), u, static_cast<int>(k)) + ";");
          em.staged[stage_in[k]] = {sp, base_of(static_cast<int>(k), rr)};
        }
        row_fwd(rr);
        em.staged.clear();
      }
      em.pop();
      body.indent--;
      body.line("}");
      body.line(r + " += (" + it + ")" + nch + " * " + std::to_string(UR * RSUB) + ";");
    } else {
    body.line("for (; " + r + " + " + std::to_string((UR - 1) * RSUB) + " < r_end; " + r + " += " +
              std::to_string(UR * RSUB) + ") {");
    body.indent++;
    em.push();
    for (int u = 0; u < UR; ++u) {
      std::string ru = em.fresh("ru");
      body.line("const " + it + " " + ru + " = " + r + " + " + std::to_string(u * RSUB) + ";");
      row(ru);
    }
    em.pop();
    body.indent--;
    body.line("}");
    }
    body.line("for (; " + r + " < r_end; " + r + " += " + std::to_string(RSUB) + ") {");
    body.indent++;
    em.push();
    row(r);
    em.pop();
    body.indent--;
    body.line("}");
    body.indent--;
    body.line("}");
  };
  // one-pass second moments (find_var2): b folds in a's pass, one level less
  const std::vector<Var2> var2 = find_var2(c, bp.level, bp.max_level);
  std::map<int, int> lvl = bp.level;
  int max_level = bp.max_level;
  std::map<int, const Var2*> var2_a, var2_b;
  for (const Var2& q : var2) {
    lvl[q.b] = lvl.at(q.a);
    var2_a[q.a] = &q;
    var2_b[q.b] = &q;
  }
  if (!var2.empty()) max_level = 1;
  // K per (pair, lane): u at reduced index 0 of the thread's columns (co/ci are
  // clamped to column 0 for threads past the last column)
  std::map<int, std::vector<std::string>> shiftK;
  for (const Var2& q : var2) {
    const Node& un = c.g.nodes[q.u];
    em.push();
    for (int l = 0; l < V; ++l) {
      const std::string v = em.value(q.u, orc_comps(em, un.dims, O, R, I, em.uni("co"), em.uni("0"), inner_ix(l)));
      const std::string k = em.fresh("shk");
      body.line("const double " + k + " = ((__float_as_uint(" + v + ") & 0x7f800000u) != 0x7f800000u) ? (double)" + v + " : 0.0;");
      shiftK[q.a].push_back(k);
    }
    em.pop();
  }
  for (int lv = 1; lv <= max_level; ++lv) {
    std::vector<int> red;
    for (int r : c.reduces)
      if (lvl.at(r) == lv) red.push_back(r);
    std::vector<std::vector<std::string>> acc(red.size(), std::vector<std::string>(V));
    for (size_t k = 0; k < red.size(); ++k) {
      const Node& rn = c.g.nodes[red[k]];
      std::string init = rn.reducer == SFX_REDUCE_SUM ? (rn.dtype == SFX_F32 ? "0.0" : "0")
                         : rn.dtype == SFX_F32        ? "sfx_bits_f(0x7fc00000)"
                         : rn.reducer == SFX_REDUCE_MAX ? "(int)0x80000000u" : "0x7fffffff";
      for (int l = 0; l < V; ++l) {
        acc[k][l] = em.fresh("acc");
        body.line(acc_t(red[k]) + " " + acc[k][l] + " = " + init + ";");
      }
    }
    stripe_pass([&](const std::string& ru) {
      Ix rix = em.uni(ru), oix = em.uni("co");
      for (int l = 0; l < V; ++l) {
        Ix iix = inner_ix(l);
        for (size_t k = 0; k < red.size(); ++k) {
          if (var2_b.count(red[k])) continue;  // folded with its first-level sum
          const Node& rn = c.g.nodes[red[k]];
          const Node& in = c.g.nodes[rn.operands[0]];
          std::string v = em.value(rn.operands[0], orc_comps(em, in.dims, O, R, I, oix, rix, iix));
          auto qa = var2_a.find(red[k]);
          if (qa != var2_a.end()) {  // shifted sums S1 (a's accumulator), S2 (b's)
            const size_t kb = std::find(red.begin(), red.end(), qa->second->b) - red.begin();
            const std::string t = em.fresh("sh");
            body.line("const double " + t + " = (double)" + v + " - " + shiftK[red[k]][l] + ";");
            body.line(acc[k][l] + " += " + t + ";");
            body.line(acc[kb][l] + " = fma(" + t + ", " + t + ", " + acc[kb][l] + ");");
            continue;
          }
          body.line(acc[k][l] + " = " + fold_fn(red[k]) + "(" + acc[k][l] + ", " + v + ");");
        }
      }
    });
    // CTA combine over row sub-streams (deterministic order), partials out
    for (size_t k = 0; k < red.size(); ++k) {
      const std::string T = acc_t(red[k]);
      const std::string sp = em.fresh("sp");
      if (NS > 0) {
        // the CTA combine reuses the (now idle) cp.async ring: reduction k's
        // [RSUB][TC] partials at k * RSUB * TC * 8 bytes; the barrier keeps
        // slower threads' last ring reads ahead of the partial writes
        if (k == 0) body.line("__syncthreads();");
        body.line(T + " (*" + sp + ")[" + fmt_i(TC) + "] = reinterpret_cast<" + T + " (*)[" + fmt_i(TC) +
                  "]>(sfx_smem + " + fmt_i(static_cast<int64_t>(k) * RSUB * TC * 8) + ");");
      } else {
        body.line("__shared__ " + T + " " + sp + "[" + std::to_string(RSUB) + "][" + fmt_i(TC) + "];");
      }
      for (int l = 0; l < V; ++l)
        body.line(sp + "[rsub][cl * " + std::to_string(V) + " + " + std::to_string(l) + "] = " + acc[k][l] + ";");
      body.line("__syncthreads();");
      body.line("if (warp == 0 && rl == 0 && cok) {");
      for (int l = 0; l < V; ++l) {
        std::string sidx = "cl * " + std::to_string(V) + " + " + std::to_string(l);
        std::string t = em.fresh("t");
        body.line("  " + T + " " + t + " = " + sp + "[0][" + sidx + "];");
        body.line("  for (int w = 1; w < " + std::to_string(RSUB) + "; ++w) " + t + " = " + fold_fn(red[k]) + "(" + t +
                  ", " + sp + "[w][" + sidx + "]);");
        body.line("  *(" + T + "*)((unsigned long long*)(ws + " + fmt_i(part_word[red[k]]) + ") + (" + it +
                  ")blockIdx.y * " + fmt_i(C) + " + c0 + " + std::to_string(l) + ") = " + t + ";");
      }
      body.line("}");
    }
    body.line("sfx_grid_barrier(ws, " + std::to_string(2 * lv - 1) + "u);");
    // the S stripe partials of each column are folded once, spread over the
    // tile's S CTAs (CTA y takes columns y, y + S, ...; its 256 threads split
    // the stripes and combine by a fixed shuffle / warp-order tree), into
    // totals[C]; a second barrier; then every thread reads its columns'
    // totals.  (Every CTA folding all S partials itself cost ~4x the data
    // pass in L2 loads: batch-norm [65536,256] 208 us.)
    for (size_t k = 0; k < red.size(); ++k) {
      const std::string T = acc_t(red[k]);
      const Node& rn = c.g.nodes[red[k]];
      std::string ident = rn.reducer == SFX_REDUCE_SUM ? (T == "double" ? "0.0" : "0")
                          : rn.dtype == SFX_F32        ? "sfx_bits_f(0x7fc00000)"
                          : rn.reducer == SFX_REDUCE_MAX ? "(int)0x80000000u" : "0x7fffffff";
      const std::string pt = "(const unsigned long long*)(ws + " + fmt_i(part_word[red[k]]) + ")";
      const std::string tt = "(unsigned long long*)(ws + " + fmt_i(tot_word[red[k]]) + ")";
      const std::string fs = em.fresh("fs");
      body.line("__shared__ " + T + " " + fs + "[" + std::to_string(WARPS) + "];");
      body.line("for (" + it + " cc = blockIdx.y; cc < " + fmt_i(TC) + "; cc += " + fmt_i(S) + ") {");
      body.line("  const " + it + " col = (" + it + ")blockIdx.x * " + fmt_i(TC) + " + cc;");
      body.line("  if (col >= " + fmt_i(C) + ") break;");
      body.line("  " + T + " a = " + ident + ";");
      body.line("  for (" + it + " s = threadIdx.x; s < " + fmt_i(S) + "; s += " + std::to_string(B) + ") a = " +
                fold_fn(red[k]) + "(a, __ldcg((const " + T + "*)(" + pt + " + s * " + fmt_i(C) + " + col)));");
      body.line(std::string("  for (int m = 16; m >= 1; m /= 2) a = ") + fold_fn(red[k]) +
                "(a, __shfl_xor_sync(0xffffffffu, a, m));");
      body.line("  if (lane == 0) " + fs + "[warp] = a;");
      body.line("  __syncthreads();");
      body.line("  if (threadIdx.x == 0) {");
      body.line("    " + T + " t = " + fs + "[0];");
      body.line("    for (int w = 1; w < " + std::to_string(WARPS) + "; ++w) t = " + std::string(fold_fn(red[k])) + "(t, " +
                fs + "[w]);");
      body.line("    *(" + T + "*)(" + tt + " + col) = t;");
      body.line("  }");
      body.line("  __syncthreads();");
      body.line("}");
    }
    body.line("sfx_grid_barrier(ws, " + std::to_string(2 * lv) + "u);");
    if (c.peer) {
      // exchange this level's totals across ranks (all reduces of the level)
      body.line("if (pn > 1) {");
      body.indent++;
      body.line("const unsigned step = launch_seq * " + std::to_string(bp.max_level) + "u + " + std::to_string(lv) + "u;");
      body.line("const long long par = step & 1u;");
      body.line("if (blockIdx.y == 0) {");
      body.line("  for (" + it + " cc = threadIdx.x; cc < " + fmt_i(TC) + "; cc += " + std::to_string(B) + ") {");
      body.line("    const " + it + " col = (" + it + ")blockIdx.x * " + fmt_i(TC) + " + cc;");
      body.line("    if (col >= " + fmt_i(C) + ") break;");
      for (size_t k = 0; k < red.size(); ++k) {
        const std::string T = acc_t(red[k]);
        body.line("    { const " + T + " v = __ldcg((const " + T + "*)((const unsigned long long*)(ws + " +
                  fmt_i(tot_word[red[k]]) + ") + col));");
        body.line("      for (int p = 0; p < pn; ++p) *(" + T + "*)((unsigned long long*)(peers[p] + poff) + ((par * " +
                  std::to_string(PMAX) + " + prank) * " + std::to_string(NR) + " + " + std::to_string(red_index[red[k]]) +
                  ") * " + fmt_i(C) + " + col) = v; }");
      }
      body.line("  }");
      body.line("  __syncthreads();");
      body.line("  if (threadIdx.x < pn) sfx_st_release_sys((unsigned*)(peers[threadIdx.x] + poff + " +
                fmt_i(pflag_byte) + ") + blockIdx.x * " + std::to_string(PMAX) + " + prank, step);");
      body.line("}");
      body.line("if (threadIdx.x < pn) sfx_peer_wait((const unsigned*)(peers[prank] + poff + " + fmt_i(pflag_byte) +
                ") + blockIdx.x * " + std::to_string(PMAX) + " + threadIdx.x, step);");
      body.line("__syncthreads();");
      body.indent--;
      body.line("}");
    }
    std::vector<int> order;  // second moments after the first-level sums they use
    for (int r : red)
      if (!var2_b.count(r)) order.push_back(r);
    for (int r : red)
      if (var2_b.count(r)) order.push_back(r);
    std::map<int, std::vector<std::string>> raw;  // fp64 totals as folded (S1 for var2 first levels)
    for (int rk : order) {
      const Node& rn = c.g.nodes[rk];
      const std::string T = acc_t(rk);
      std::vector<std::string> tv(V);
      for (int l = 0; l < V; ++l) {
        tv[l] = em.fresh("tot");
        body.line(T + " " + tv[l] + " = __ldcg((const " + T + "*)((const unsigned long long*)(ws + " +
                  fmt_i(tot_word[rk]) + ") + (cok ? c0 : 0) + " + std::to_string(l) + "));");
      }
      raw[rk] = tv;
      if (var2_a.count(rk))  // A = N·K + S1
        for (int l = 0; l < V; ++l) {
          const std::string f = em.fresh("tot");
          body.line("const double " + f + " = " + fmt_i(R) + ".0 * " + shiftK[rk][l] + " + " + tv[l] + ";");
          tv[l] = f;
        }
      auto qb = var2_b.find(rk);
      if (qb != var2_b.end()) {  // b = S2 - 2δ·S1 + N·δ², δ = m - K (m: the graph's fp32 mean)
        const Var2& q = *qb->second;
        const Node& mbn = c.g.nodes[q.mb];
        em.push();
        for (int l = 0; l < V; ++l) {
          const std::string m = em.value(q.mb, orc_comps(em, mbn.dims, O, R, I, em.uni("co"), em.uni("0"), inner_ix(l)));
          const std::string dl = em.fresh("dl"), f = em.fresh("tot");
          body.line("const double " + dl + " = (double)" + m + " - " + shiftK[q.a][l] + ";");
          // non-finite mean (an inf / NaN in the column, or an fp32 overflow of its
          // sum): Σ (u - m)² as the two-level form gets it — NaN for a NaN mean or when
          // some u equals the infinite mean (S1 not finite), else +inf
          body.line("const double " + f + " = ((__float_as_uint(" + m + ") & 0x7f800000u) != 0x7f800000u) ? " + tv[l] + " - 2.0 * " + dl + " * " +
                    raw[q.a][l] + " + " + fmt_i(R) + ".0 * " + dl + " * " + dl + " : (" + m + " != " + m +
                    " || !(fabs(" + raw[q.a][l] + ") <= 1.7976931348623157e308)) ? (double)(" + m + " - " + m + ") : (double)(" + m +
                    " * " + m + ");");
          tv[l] = f;
        }
        em.pop();
      }
      if (c.peer) {  // the ranks' totals, in rank order (identical on every rank)
        body.line("if (pn > 1) {");
        body.line("  const long long par = (launch_seq * " + std::to_string(bp.max_level) + "u + " + std::to_string(lv) +
                  "u) & 1u;");
        body.line("  const unsigned long long* xs = (const unsigned long long*)(peers[prank] + poff) + (par * " +
                  std::to_string(PMAX) + " * " + std::to_string(NR) + " + " + std::to_string(red_index[rk]) + ") * " +
                  fmt_i(C) + " + (cok ? c0 : 0);");
        for (int l = 0; l < V; ++l) {
          body.line("  " + tv[l] + " = __ldcv((const " + T + "*)(xs + " + std::to_string(l) + "));");
          body.line("  for (int q = 1; q < pn; ++q) " + tv[l] + " = " + fold_fn(rk) + "(" + tv[l] + ", __ldcv((const " +
                    T + "*)(xs + (long long)q * " + std::to_string(NR) + " * " + fmt_i(C) + " + " + std::to_string(l) +
                    ")));");
        }
        body.line("}");
      }
      if (T == "double")
        for (int l = 0; l < V; ++l) {
          std::string f = em.fresh("tot");
          body.line("const float " + f + " = (float)" + tv[l] + ";");
          tv[l] = f;
        }
      if (rn.reducer != SFX_REDUCE_SUM && rn.dtype == SFX_F32) {
        const Node& in = c.g.nodes[rn.operands[0]];
        for (int l = 0; l < V; ++l) {
          em.push();
          Ix iix = inner_ix(l);
          std::string f0 = em.value(rn.operands[0], orc_comps(em, in.dims, O, R, I, em.uni("co"), em.uni("0"), iix));
          body.line(tv[l] + " = sfx_fold_first(" + f0 + ", " + tv[l] + ");");
          em.pop();
        }
      }
      total[rk] = tv;
    }
  }
  // final pass: element roots; column roots from stripe 0
  std::vector<int> full_roots, col_roots;
  for (int r : c.p.roots) (c.g.nodes[r].numel() == O * R * I ? full_roots : col_roots).push_back(r);
  if (!full_roots.empty())
    stripe_pass([&](const std::string& ru) {
      Ix rix = em.uni(ru), oix = em.uni("co");
      std::vector<std::vector<std::string>> fv(full_roots.size(), std::vector<std::string>(V));
      std::vector<std::string> faddr(full_roots.size());
      std::vector<bool> fvec(full_roots.size(), V == 4);
      std::vector<std::vector<std::string>> fad(full_roots.size(), std::vector<std::string>(V));
      for (int l = 0; l < V; ++l) {
        Ix iix = inner_ix(l);
        for (size_t k = 0; k < full_roots.size(); ++k) {
          std::vector<Ix> comps = orc_comps(em, c.g.nodes[full_roots[k]].dims, O, R, I, oix, rix, iix);
          fv[k][l] = em.value(full_roots[k], comps);
          Ix L = em.linearize(comps, c.g.nodes[full_roots[k]].dims);
          fad[k][l] = L.e;
          if (l == 0) {
            if (L.kind == IX_PLUS) faddr[k] = L.base;
            else fvec[k] = false;
          }
        }
      }
      for (size_t k = 0; k < full_roots.size(); ++k) {
        std::string out = "out" + std::to_string(root_slot(c, full_roots[k]));
        if (fvec[k])
          body.line("sfx_st4(" + out + " + " + faddr[k] + ", " + fv[k][0] + ", " + fv[k][1] + ", " + fv[k][2] + ", " +
                    fv[k][3] + ");");
        else
          for (int l = 0; l < V; ++l) body.line(out + "[" + fad[k][l] + "] = " + fv[k][l] + ";");
      }
    });
  if (!col_roots.empty()) {
    body.line("if (blockIdx.y == 0 && warp == 0 && rl == 0 && cok) {");
    body.indent++;
    em.push();
    for (int r : col_roots) {
      for (int l = 0; l < V; ++l) {
        em.lane = l;
        Ix col = V == 1 ? em.uni("c0") : em.lane_plus("c0");
        std::string v = em.value(r, em.from_linear(col, c.g.nodes[r].dims));
        body.line("out" + std::to_string(root_slot(c, r)) + "[c0 + " + std::to_string(l) + "] = " + v + ";");
      }
    }
    em.pop();
    body.indent--;
    body.line("}");
  }
  if (c.peer)  // the last CTA out also advances the launch sequence
    body.line("if (threadIdx.x == 0 && atomicAdd(ws + 1, 1u) == gridDim.x * gridDim.y - 1u) { ws[0] = 0u; ws[1] = 0u; "
              "ws[2] = launch_seq + 1u; }");
  else
    body.line("sfx_grid_exit(ws);");
  ks.code = assemble(sig, body);
  ks.block = B;
  ks.grid_x = tiles;
  ks.grid_y = S;
  ks.vector_width = V;
  ks.note = "outer=" + std::to_string(O) + " reduced=" + std::to_string(R) + " inner=" + std::to_string(I) +
            " tiles=" + std::to_string(tiles) + " stripes=" + std::to_string(S) + " levels=" +
            std::to_string(max_level) + " (grid barriers, cooperative launch)" +
            (var2.empty() ? "" : ", " + std::to_string(var2.size()) + " second moment(s) in the first pass") +
            (NS > 0 ? ", cp.async ring " + std::to_string(NS) + " x " + std::to_string(UR) + " rows" : "");
  return ks;
}

// Channel statistics broadcast back over [A | K | B] (reduce A and B, keep K:
// batch-norm over NCHW).  A CTA tile is one channel; S stripes of its A·B/V
// vectors (V = 4 along the contiguous B block when B % 4 == 0).  Per level: a
// pass over the stripe (fp64 accumulators, lanes folded together; the
// variance as shifted sums in the mean's pass, find_var2), a warp-order CTA
// combine, then with S > 1 partials to the workspace, one grid barrier and every
// CTA of the channel folding the S partials in stripe order (identical totals;
// cooperative launch); with S == 1 (K >= 148 channels) no grid barrier at all.
// Passes alternate direction (the re-read starts on the vectors still in L2).
KernelSource lower_colbc_split(const Ctx& c, const SplitPlan& sp, const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "colbc";
  ks.entry = "sfx_colbc_" + c.name;
  fill_common(c, ks);
  const int64_t A = sp.A, K = sp.K, B = sp.B;
  const int V = (B % 4 == 0) ? 4 : 1;
  const int64_t BV = B / V, NV = A * BV;  // vectors per channel
  const int WARPS = 8, T = WARPS * 32;
  const int ctas_per_sm = o.pipe_ctas_per_sm > 0 ? std::min(o.pipe_ctas_per_sm, 8) : 2;
  int64_t S = o.rows_per_cta > 0 ? o.rows_per_cta : std::max<int64_t>(1, kNumSMs * ctas_per_sm / K);
  S = std::max<int64_t>(1, std::min<int64_t>(S, NV / (4 * T)));
  if (S > 1 && K * S > int64_t{kNumSMs} * ctas_per_sm) S = std::max<int64_t>(1, kNumSMs * ctas_per_sm / K);
  // a channel per CTA leaves SMs unevenly loaded when K is not a multiple of
  // the SM count (256 channels on 148 SMs: 108 SMs carry two): from 37 channels
  // up, a thread-block cluster of CS CTAs takes each channel instead (>= 4
  // clusters' worth of CTAs per SM), the CTAs combining their partials through
  // distributed shared memory — no grid barrier.  pipe_stages = 1: one CTA per
  // channel (A/B)
  int CS = 1;
  if (K * 8 >= int64_t{kNumSMs} * 2 && o.pipe_stages != 1 && o.rows_per_cta <= 0) {
    S = 1;
    while (CS < 8 && K * CS < int64_t{kNumSMs} * 4 && NV / (CS * 2) >= 4 * T) CS *= 2;
  }
  const int64_t RS = (NV + S * CS - 1) / (S * CS);
  const int UR = o.items_per_thread > 0 ? std::min(o.items_per_thread, 16) : 8;
  std::vector<Var2> var2 = find_var2(c, sp.level, sp.max_level);
  std::map<int, int> lvl = sp.level;
  int max_level = sp.max_level;
  std::map<int, const Var2*> var2_a, var2_b;
  for (const Var2& q : var2) {
    lvl[q.b] = lvl.at(q.a);
    var2_a[q.a] = &q;
    var2_b[q.b] = &q;
  }
  if (!var2.empty()) max_level = 1;
  Emitter em(c.g, c.p, V, c.wide);
  em.rcp_reduced_divisors = rcp_divisors();
  std::string sig = signature(c, em, ks.entry, T, ctas_per_sm);
  if (CS > 1) {
    const std::string gv = "__global__ void ";
    sig.insert(sig.find(gv) + gv.size(), "__cluster_dims__(" + std::to_string(CS) + ", 1, 1) ");
  }
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  // workspace: barrier counters (64 words), then per reduce partials[S][K] (8-byte slots)
  std::map<int, int64_t> part_word;
  int64_t words = 64;
  for (int r : c.reduces) {
    part_word[r] = words;
    words += S * K * 2;
  }
  if (S > 1) {
    ks.workspace_bytes = words * 4;
    ks.cooperative = true;
  }
  body.line("const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;");
  if (CS > 1) {
    body.line("const " + it + " kc = (" + it + ")blockIdx.x / " + std::to_string(CS) + ";");
    body.line("const " + it + " v_begin = (" + it + ")(blockIdx.x % " + std::to_string(CS) + ") * " + fmt_i(RS) + ";");
  } else {
    body.line("const " + it + " kc = (" + it + ")blockIdx.x;");
    body.line("const " + it + " v_begin = (" + it + ")blockIdx.y * " + fmt_i(RS) + ";");
  }
  body.line("const " + it + " v_end = min((" + it + ")" + fmt_i(NV) + ", v_begin + " + fmt_i(RS) + ");");
  const Ix kix = em.uni("kc");
  // element (a, kc, b) of a node of `dims`; vector v = a * BV + b / V
  auto elem = [&](const std::vector<int64_t>& dims, const std::string& a, const std::string& b0, int l) {
    em.lane = l;
    Ix bix = V == 1 ? em.uni(b0) : em.lane_plus(b0);
    return orc_comps(em, dims, A, K, B, em.uni(a), kix, bix);
  };
  std::map<int, std::string> total;
  em.resolve = [&](int node, const std::vector<Ix>&) -> std::string {
    auto f = total.find(node);
    if (f == total.end()) {
      if (c.g.nodes[node].op == SFX_OP_REDUCE && !degenerate_reduce(c.g, c.g.nodes[node]))
        throw Error(SFX_ERR_INVALID, "internal: reduction used before it is combined");
      return "";
    }
    return f->second;
  };
  // K per second-moment pair: u at (0, kc, 0); 0 when not finite
  std::map<int, std::string> shiftK;
  for (const Var2& q : var2) {
    em.push();
    const std::string v = em.value(q.u, elem(c.g.nodes[q.u].dims, "0", "0", 0));
    const std::string k = em.fresh("shk");
    body.line("const double " + k + " = ((__float_as_uint(" + v + ") & 0x7f800000u) != 0x7f800000u) ? (double)" + v +
              " : 0.0;");
    shiftK[q.a] = k;
    em.pop();
  }
  int pass_no = 0;
  // a pass over this CTA's vectors: UR per thread per iteration (loads in flight together)
  auto stripe_pass = [&](const std::function<void(const std::string&, const std::string&)>& vec) {
    const bool rev = pass_no++ % 2 == 1;
    auto one = [&](const std::string& vf) {
      std::string vv = vf;
      if (rev) {
        vv = em.fresh("vr");
        body.line("const " + it + " " + vv + " = v_begin + v_end - 1 - (" + vf + ");");
      }
      const std::string a = em.fresh("a"), b0 = em.fresh("b");
      body.line("const " + it + " " + a + " = " + vv + " / " + fmt_i(BV) + ";");
      body.line("const " + it + " " + b0 + " = (" + vv + " - " + a + " * " + fmt_i(BV) + ") * " + std::to_string(V) + ";");
      vec(a, b0);
    };
    const std::string v = em.fresh("v");
    body.line(it + " " + v + " = v_begin + threadIdx.x;");
    body.line("for (; " + v + " + " + std::to_string((UR - 1) * T) + " < v_end; " + v + " += " + std::to_string(UR * T) +
              ") {");
    body.indent++;
    em.push();
    for (int u = 0; u < UR; ++u) {
      const std::string vu = em.fresh("vu");
      body.line("const " + it + " " + vu + " = " + v + " + " + std::to_string(u * T) + ";");
      one(vu);
    }
    em.pop();
    body.indent--;
    body.line("}");
    body.line("for (; " + v + " < v_end; " + v + " += " + std::to_string(T) + ") {");
    body.indent++;
    em.push();
    one(v);
    em.pop();
    body.indent--;
    body.line("}");
  };
  for (int lv = 1; lv <= max_level; ++lv) {
    std::vector<int> red;
    for (int r : c.reduces)
      if (lvl.at(r) == lv) red.push_back(r);
    std::vector<std::string> acc(red.size());
    for (size_t k = 0; k < red.size(); ++k) {
      acc[k] = em.fresh("acc");
      body.line("double " + acc[k] + " = 0.0;");
    }
    stripe_pass([&](const std::string& a, const std::string& b0) {
      for (int l = 0; l < V; ++l) {
        for (size_t k = 0; k < red.size(); ++k) {
          if (var2_b.count(red[k])) continue;  // folded with its first-level sum
          const Node& rn = c.g.nodes[red[k]];
          std::string v = em.value(rn.operands[0], elem(c.g.nodes[rn.operands[0]].dims, a, b0, l));
          auto qa = var2_a.find(red[k]);
          if (qa != var2_a.end()) {
            const size_t kb = std::find(red.begin(), red.end(), qa->second->b) - red.begin();
            const std::string t = em.fresh("sh");
            body.line("const double " + t + " = (double)" + v + " - " + shiftK[red[k]] + ";");
            body.line(acc[k] + " += " + t + ";");
            body.line(acc[kb] + " = fma(" + t + ", " + t + ", " + acc[kb] + ");");
            continue;
          }
          body.line(acc[k] + " += (double)" + v + ";");
        }
      }
    });
    // CTA combine: warp shuffle tree, then the warps in order
    for (size_t k = 0; k < red.size(); ++k) {
      for (int m = 16; m >= 1; m /= 2)
        body.line(acc[k] + " += __shfl_xor_sync(0xffffffffu, " + acc[k] + ", " + std::to_string(m) + ");");
      const std::string sm = em.fresh("wsm");
      body.line("__shared__ double " + sm + "[" + std::to_string(WARPS) + "];");
      body.line("if (lane == 0) " + sm + "[warp] = " + acc[k] + ";");
      body.line("__syncthreads();");
      body.line(acc[k] + " = " + sm + "[0];");
      body.line("for (int w = 1; w < " + std::to_string(WARPS) + "; ++w) " + acc[k] + " += " + sm + "[w];");
      if (S > 1)
        body.line("if (threadIdx.x == 0) *(double*)((unsigned long long*)(ws + " + fmt_i(part_word[red[k]]) +
                  ") + (" + it + ")blockIdx.y * " + fmt_i(K) + " + kc) = " + acc[k] + ";");
    }
    if (CS > 1) {
      // cluster combine: every CTA folds the CS partials in rank order (identical
      // totals); the second cluster barrier keeps every CTA's shared memory alive
      // until its peers have read it
      const std::string xp = em.fresh("xp"), xr = em.fresh("xr");
      body.line("__shared__ double " + xp + "[" + std::to_string(red.size()) + "], " + xr + "[" +
                std::to_string(red.size()) + "];");
      for (size_t k = 0; k < red.size(); ++k)
        body.line("if (threadIdx.x == 0) " + xp + "[" + std::to_string(k) + "] = " + acc[k] + ";");
      body.line("sfx_cluster_sync();");
      body.line("if (warp == 0) {");
      for (size_t k = 0; k < red.size(); ++k) {
        body.line("  { const double v = lane < " + std::to_string(CS) + " ? sfx_dsmem_ld(&" + xp + "[" +
                  std::to_string(k) + "], (unsigned)lane) : 0.0;");
        body.line("    double a = __shfl_sync(0xffffffffu, v, 0);");
        body.line("    for (int r = 1; r < " + std::to_string(CS) + "; ++r) a += __shfl_sync(0xffffffffu, v, r);");
        body.line("    if (lane == 0) " + xr + "[" + std::to_string(k) + "] = a; }");
      }
      body.line("}");
      body.line("sfx_cluster_sync();");
      for (size_t k = 0; k < red.size(); ++k) body.line(acc[k] + " = " + xr + "[" + std::to_string(k) + "];");
    }
    if (S > 1) {
      body.line("sfx_grid_barrier(ws, " + std::to_string(lv) + "u);");
      // every CTA of the channel folds its S partials in stripe order (identical totals)
      for (size_t k = 0; k < red.size(); ++k) {
        body.line(acc[k] + " = 0.0;");
        body.line("for (int s = 0; s < " + fmt_i(S) + "; ++s) " + acc[k] + " += __ldcg((const double*)((const unsigned long long*)(ws + " +
                  fmt_i(part_word[red[k]]) + ") + (" + it + ")s * " + fmt_i(K) + " + kc));");
      }
    }
    std::vector<size_t> order;
    for (size_t k = 0; k < red.size(); ++k)
      if (!var2_b.count(red[k])) order.push_back(k);
    for (size_t k = 0; k < red.size(); ++k)
      if (var2_b.count(red[k])) order.push_back(k);
    for (size_t k : order) {
      std::string fin = em.fresh("tot");
      if (var2_a.count(red[k])) {  // A = N·K + S1
        body.line("const float " + fin + " = (float)(" + fmt_i(A * B) + ".0 * " + shiftK[red[k]] + " + " + acc[k] + ");");
      } else if (var2_b.count(red[k])) {  // b = S2 - 2δ·S1 + N·δ²; a non-finite mean as in Σ (u - m)²
        const Var2& q = *var2_b.at(red[k]);
        const size_t ka = std::find(red.begin(), red.end(), q.a) - red.begin();
        em.push();
        const std::string m = em.value(q.mb, elem(c.g.nodes[q.mb].dims, "0", "0", 0));
        em.pop();
        const std::string dl = em.fresh("dl");
        body.line("const double " + dl + " = (double)" + m + " - " + shiftK[q.a] + ";");
        body.line("const float " + fin + " = (float)(((__float_as_uint(" + m + ") & 0x7f800000u) != 0x7f800000u) ? " +
                  acc[k] + " - 2.0 * " + dl + " * " + acc[ka] + " + " + fmt_i(A * B) + ".0 * " + dl + " * " + dl +
                  " : (" + m + " != " + m + " || !(fabs(" + acc[ka] + ") <= 1.7976931348623157e308)) ? (double)(" + m +
                  " - " + m + ") : (double)(" + m + " * " + m + "));");
      } else {
        body.line("const float " + fin + " = (float)" + acc[k] + ";");
      }
      total[red[k]] = fin;
    }
  }
  // final pass: element roots; channel roots by stripe 0
  std::vector<int> full_roots, chan_roots;
  for (int r : c.p.roots) (c.g.nodes[r].numel() == A * K * B ? full_roots : chan_roots).push_back(r);
  if (!full_roots.empty())
    stripe_pass([&](const std::string& a, const std::string& b0) {
      std::vector<std::vector<std::string>> fv(full_roots.size(), std::vector<std::string>(V));
      std::vector<std::vector<std::string>> fad(full_roots.size(), std::vector<std::string>(V));
      std::vector<std::string> base(full_roots.size());
      std::vector<bool> fvec(full_roots.size(), V == 4);
      for (int l = 0; l < V; ++l)
        for (size_t k = 0; k < full_roots.size(); ++k) {
          std::vector<Ix> comps = elem(c.g.nodes[full_roots[k]].dims, a, b0, l);
          fv[k][l] = em.value(full_roots[k], comps);
          Ix L = em.linearize(comps, c.g.nodes[full_roots[k]].dims);
          fad[k][l] = L.e;
          if (l == 0) {
            if (L.kind == IX_PLUS) base[k] = L.base;
            else fvec[k] = false;
          }
        }
      for (size_t k = 0; k < full_roots.size(); ++k) {
        const std::string out = "out" + std::to_string(root_slot(c, full_roots[k]));
        if (fvec[k])
          body.line("sfx_st4(" + out + " + " + base[k] + ", " + fv[k][0] + ", " + fv[k][1] + ", " + fv[k][2] + ", " +
                    fv[k][3] + ");");
        else
          for (int l = 0; l < V; ++l) body.line(out + "[" + fad[k][l] + "] = " + fv[k][l] + ";");
      }
    });
  if (!chan_roots.empty()) {
    body.line(std::string("if (") + (CS > 1 ? "v_begin == 0" : "blockIdx.y == 0") + " && threadIdx.x == 0) {");
    body.indent++;
    em.push();
    em.lane = 0;
    for (int r : chan_roots) {
      std::string v = em.value(r, em.from_linear(kix, c.g.nodes[r].dims));
      body.line("out" + std::to_string(root_slot(c, r)) + "[kc] = " + v + ";");
    }
    em.pop();
    body.indent--;
    body.line("}");
  }
  if (S > 1) body.line("sfx_grid_exit(ws);");
  ks.code = assemble(sig, body);
  ks.block = T;
  ks.grid_x = K * CS;
  ks.grid_y = S;
  ks.cluster = CS;
  ks.vector_width = V;
  ks.note = "split A=" + std::to_string(A) + " channels=" + std::to_string(K) + " B=" + std::to_string(B) +
            " stripes=" + std::to_string(S) + " levels=" + std::to_string(max_level) +
            (S > 1 ? " (grid barriers, cooperative launch)"
             : CS > 1 ? " (a cluster of " + std::to_string(CS) + " CTAs per channel, DSMEM combine, no grid barrier)"
                      : " (one CTA per channel, no grid barrier)") +
            (var2.empty() ? "" : ", " + std::to_string(var2.size()) + " second moment(s) in the first pass");
  return ks;
}

}  // namespace lw
}  // namespace sfx
