// kLoop (map) template and the shared-memory-tiled transpose variant.
#include "lower_impl.hpp"

namespace sfx {
namespace lw {

// ---- MAP -----------------------------------------------------------------------

bool analyze_map(const Ctx& c, std::string* why) {
  if (!c.dots.empty()) return *why = "group contains a matmul", false;
  if (!c.reduces.empty()) return *why = "group has reductions", false;
  return true;
}

std::set<int> row_local_inputs(const Ctx& c, const RowPlan& rp);

KernelSource lower_map(const Ctx& c, const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "map";
  ks.entry = "sfx_map_" + c.name;
  fill_common(c, ks);
  const int B = 256;
  // shape classes: roots with identical dims share one loop (and their CSE)
  std::map<std::vector<int64_t>, std::vector<int>> classes;
  for (int r : c.p.roots) classes[c.g.nodes[r].dims].push_back(r);
  int vmax = 1;
  int64_t max_items = 1;
  std::vector<std::pair<int, int64_t>> vw;  // per class: V, items
  for (auto& [dims, roots] : classes) {
    int64_t n = prod(dims, 0, dims.size());
    int V = (!dims.empty() && dims.back() % 4 == 0) ? 4 : 1;
    vw.push_back({V, n / V});
    vmax = std::max(vmax, V);
    max_items = std::max(max_items, n / V);
  }
  Code body;
  // items (V-element vectors) per thread: several independent 128-bit loads in
  // flight per thread on large streams; consecutive threads stay consecutive
  int U = o.items_per_thread > 0 ? o.items_per_thread
          : max_items >= int64_t{kNumSMs} * 8 * B * 4 ? 4
          : max_items >= int64_t{kNumSMs} * 8 * B * 2 ? 2 : 1;
  U = std::max(1, std::min(U, 8));
  // host streaming over the root's leading dim (one shape class only)
  const bool stream = o.host_stream && classes.size() == 1 && !classes.begin()->first.empty() &&
                      classes.begin()->first[0] > 1;
  if (stream) {
    const std::vector<int64_t>& dims = classes.begin()->first;
    RowPlan sp;
    sp.R = dims[0];
    sp.C = prod(dims, 1, dims.size());
    ks.stream_R = sp.R;
    ks.stream_C = sp.C;
    ks.stream_cta_elems = int64_t{B} * U * vw[0].first;
    ks.stream_unit = ks.stream_cta_elems / gcd64(ks.stream_cta_elems, sp.C);
    std::set<int> loc = row_local_inputs(c, sp);
    ks.stream_inputs.assign(loc.begin(), loc.end());
  }
  // one emitter per class (lane count differs)
  std::string sig;
  {
    Emitter probe(c.g, c.p, 1, c.wide);
    sig = signature(c, probe, ks.entry, B, 0, stream);
  }
  std::string idx_t = c.wide ? "long long" : "int";
  if (stream)
    emit_stream_gate(body, "(long long)blockIdx.x * " + fmt_i(ks.stream_cta_elems), ks.stream_cta_elems,
                     ks.stream_R * ks.stream_C);
  body.line("const " + idx_t + " t0 = (" + idx_t + ")blockIdx.x * " + std::to_string(B * U) + " + threadIdx.x;");
  size_t ci = 0;
  for (auto& [dims, roots] : classes) {
    auto [V, items] = vw[ci++];
    Emitter em(c.g, c.p, V, c.wide);
    signature(c, em, ks.entry, B, 0, stream);
    em.code = &body;
    auto emit_item = [&](const std::string& it) {
      em.push();
      std::string base = V == 1 ? it : em.ivar(Emitter::imul(it, V));
      std::vector<std::vector<std::string>> vals(roots.size(), std::vector<std::string>(V));
      for (int lane = 0; lane < V; ++lane) {
        em.lane = lane;
        Ix L = V == 1 ? em.uni(base) : em.lane_plus(base);
        for (size_t k = 0; k < roots.size(); ++k) {
          std::vector<Ix> comps = em.from_linear(L, c.g.nodes[roots[k]].dims);
          vals[k][lane] = em.value(roots[k], comps);
        }
      }
      for (size_t k = 0; k < roots.size(); ++k) {
        std::string out = "out" + std::to_string(root_slot(c, roots[k]));
        if (V == 4)
          body.line("sfx_st4(" + out + " + " + base + ", " + vals[k][0] + ", " + vals[k][1] + ", " +
                    vals[k][2] + ", " + vals[k][3] + ");");
        else
          body.line(out + "[" + base + "] = " + vals[k][0] + ";");
      }
      em.pop();
    };
    auto item_var = [&](int u) { return "t" + std::to_string(ci) + "_" + std::to_string(u); };
    if (U > 1) {
      // full tiles: U unguarded items (loads of all items can issue together)
      body.line("if (t0 + " + fmt_i(static_cast<int64_t>(U - 1) * B) + " < " + fmt_i(items) + ") {");
      body.indent++;
      for (int u = 0; u < U; ++u) {
        body.line("const " + idx_t + " " + item_var(u) + " = t0 + " + std::to_string(u * B) + ";");
        emit_item(item_var(u));
      }
      body.indent--;
      body.line("} else {");
      body.indent++;
    }
    for (int u = 0; u < U; ++u) {
      body.line("{");
      body.indent++;
      body.line("const " + idx_t + " " + item_var(u) + " = t0 + " + std::to_string(u * B) + ";");
      body.line("if (" + item_var(u) + " < " + fmt_i(items) + ") {");
      body.indent++;
      emit_item(item_var(u));
      body.indent--;
      body.line("}");
      body.indent--;
      body.line("}");
    }
    if (U > 1) {
      body.indent--;
      body.line("}");
    }
  }
  if (stream) emit_stream_done(body, "(long long)blockIdx.x * " + fmt_i(ks.stream_cta_elems));
  ks.code = assemble(sig, body);
  ks.block = B;
  ks.grid_x = (max_items + int64_t{B} * U - 1) / (int64_t{B} * U);
  ks.vector_width = vmax;
  ks.note = "kLoop over " + std::to_string(classes.size()) + " root shape class(es), " + std::to_string(U) +
            " vector item(s)/thread";
  return ks;
}

// ---- MAP with shared-memory-tiled transposes ---------------------------------------

// Symbolic index walk from the root: every dimension of every reached node is
// labelled with the root axes it is indexed by, as row-major components
// (axis, extent) — one component for a plain axis, several where a reshape
// merged root axes into one dimension (BERT's [T, Hd] = [B*S, NH*D] feeding
// a head transpose), none for a unit dimension — or kUnknown when a reshape
// splits an axis or an op mixes indices.  Returns, per external, the set of
// distinct labellings it is read with.

bool labels_known(const Labels& t) {
  for (const DimLabel& d : t)
    for (auto& c : d)
      if (c.first == kUnknown) return false;
  return true;
}

std::map<int, std::set<Labels>> index_labels(const Ctx& c, int root) {
  std::map<int, std::set<Labels>> ext;
  std::set<std::pair<int, Labels>> seen;
  auto unknown = [](int rank) { return Labels(rank, DimLabel{{kUnknown, 0}}); };
  std::function<void(int, const Labels&)> walk = [&](int n, const Labels& t) {
    if (!seen.insert({n, t}).second) return;
    const Node& m = c.g.nodes[n];
    if (!c.p.is_member(n)) {
      if (!m.is_splat()) ext[n].insert(t);
      return;
    }
    switch (m.op) {
      case SFX_OP_ELEMENTWISE:
        for (int o : m.operands) walk(o, t);
        return;
      case SFX_OP_TRANSPOSE: {
        Labels in(t.size());
        for (size_t i = 0; i < t.size(); ++i) in[m.perm[i]] = t[i];
        walk(m.operands[0], in);
        return;
      }
      case SFX_OP_BROADCAST: {
        Labels in(m.dim_map.size());
        for (size_t j = 0; j < m.dim_map.size(); ++j) in[j] = t[m.dim_map[j]];
        walk(m.operands[0], in);
        return;
      }
      case SFX_OP_RESHAPE:
      case SFX_OP_BITCAST: {
        // row-major: the flattened component sequence is shared; regroup it
        // into the operand's dims without splitting a component
        const Node& in = c.g.nodes[m.operands[0]];
        if (!labels_known(t)) return walk(m.operands[0], unknown(in.rank()));
        DimLabel seq;
        for (const DimLabel& d : t) seq.insert(seq.end(), d.begin(), d.end());
        Labels r(in.rank());
        size_t k = 0;
        for (int i = 0; i < in.rank(); ++i) {
          int64_t need = in.dims[i], have = 1;
          while (have < need && k < seq.size()) {
            have *= seq[k].second;
            r[i].push_back(seq[k++]);
          }
          if (have != need) return walk(m.operands[0], unknown(in.rank()));
        }
        walk(m.operands[0], r);
        return;
      }
      default: {
        for (int o : m.operands) walk(o, unknown(c.g.nodes[o].rank()));
        return;
      }
    }
  };
  Labels t;
  const Node& rn = c.g.nodes[root];
  for (int i = 0; i < rn.rank(); ++i) t.push_back(rn.dims[i] == 1 ? DimLabel{} : DimLabel{{i, rn.dims[i]}});
  walk(root, t);
  return ext;
}


// A map group whose (single-shape) roots read a streamed input whose innermost
// dimension is indexed by a root axis other than the root's innermost: the
// naive kLoop would read it with a stride.  Tile (a, b) through shared memory.
bool analyze_tiled(const Ctx& c, TilePlan* tp) {
  if (!c.reduces.empty() || !c.dots.empty()) return false;
  const std::vector<int64_t>& dims = c.g.nodes[c.p.roots[0]].dims;
  for (int r : c.p.roots)
    if (c.g.nodes[r].dims != dims) return false;
  const int n = static_cast<int>(dims.size());
  if (n < 2) return false;
  tp->a = n - 1;
  std::map<int, int> votes;
  std::map<int, Emitter::Tile> cand;
  std::map<int, int> bof;
  std::map<int, std::set<Labels>> merged;
  for (int r : c.p.roots)
    for (auto& [e, ts] : index_labels(c, r)) merged[e].insert(ts.begin(), ts.end());
  for (auto& [e, ts] : merged) {
    const Node& en = c.g.nodes[e];
    if (ts.size() != 1 || en.rank() < 1 || en.numel() * 4 < (1 << 20)) continue;
    const Labels& t = *ts.begin();
    if (!labels_known(t) || t.back().empty()) continue;
    const std::pair<int, int64_t>& fastest = t.back().back();
    if (fastest.first == tp->a) continue;  // already coalesced along the root's innermost axis
    Emitter::Tile tile;
    tile.jb = en.rank() - 1;
    tile.mb = t.back().size() > 1 ? fastest.second : 0;
    bool found = false;
    for (int d = 0; d < en.rank() && !found; ++d) {
      int64_t stride = 1;
      for (int q = static_cast<int>(t[d].size()) - 1; q >= 0; --q) {
        if (t[d][q].first == tp->a) {
          tile.ja = d;
          tile.sa = stride;
          tile.ma = t[d].size() > 1 ? t[d][q].second : 0;
          found = true;
          break;
        }
        stride *= t[d][q].second;
      }
    }
    if (!found || tile.ja == tile.jb) continue;
    cand[e] = tile;
    bof[e] = fastest.first;
    votes[fastest.first]++;
  }
  if (votes.empty()) return false;
  tp->b = std::max_element(votes.begin(), votes.end(), [](auto& x, auto& y) { return x.second < y.second; })->first;
  for (auto& [e, tile] : cand)
    if (bof[e] == tp->b) {
      tp->inputs[e] = tile;
      tp->labels[e] = *merged[e].begin();
    }
  return !tp->inputs.empty();
}

// The vectorised tiled transpose: 64 x 64 tiles over root axes (a = root
// innermost, b = the tiled inputs' innermost), 256 threads.
//   load:    each thread LDG.128s 4 consecutive b of one a-row (16 threads per
//            row, 4 passes) and STS.128s them into the row's XOR-swizzled
//            16-byte chunk (conflict-free: 8 threads of a phase hit 8 chunks);
//   compute: a warp covers 8 a-vectors (32 consecutive a) x 4 b; each thread
//            reads its 4 a-values (4 LDS.32, the swizzle puts the warp's 8 rows
//            x 4 b on 32 distinct banks), evaluates the roots for 4 lanes and
//            STG.128s them — 4 full 128-byte lines per warp store.
KernelSource lower_map_tiled_v4(const Ctx& c, const TilePlan& tp, const sfx_compile_opts& o) {
  (void)o;
  KernelSource ks;
  ks.strategy = "map";
  ks.entry = "sfx_mapt_" + c.name;
  fill_common(c, ks);
  const std::vector<int64_t>& dims = c.g.nodes[c.p.roots[0]].dims;
  const int n = static_cast<int>(dims.size());
  const int a = tp.a, b = tp.b;
  const int64_t na = dims[a], nb = dims[b];
  const int TT = 64;
  const int64_t nta = (na + TT - 1) / TT, ntb = (nb + TT - 1) / TT;
  std::vector<int64_t> rest_dims;
  std::vector<int> rest_axes;
  for (int i = 0; i < n; ++i)
    if (i != a && i != b) rest_dims.push_back(dims[i]), rest_axes.push_back(i);
  const int64_t nrest = prod(rest_dims, 0, rest_dims.size());
  Emitter em(c.g, c.p, 4, c.wide);
  std::string sig = signature(c, em, ks.entry, 256);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  body.line("const int tid = threadIdx.x;");
  body.line(it + " tix = blockIdx.x;");
  body.line("const " + it + " a0 = (tix % " + fmt_i(nta) + ") * " + std::to_string(TT) + "; tix /= " + fmt_i(nta) + ";");
  body.line("const " + it + " b0 = (tix % " + fmt_i(ntb) + ") * " + std::to_string(TT) + "; tix /= " + fmt_i(ntb) + ";");
  body.line("const " + it + " rest = tix;");
  std::vector<Ix> rest = em.from_linear(em.uni("rest"), rest_dims);
  int ti = 0;
  for (auto& [e, tile] : tp.inputs) {
    const Node& en = c.g.nodes[e];
    Emitter::Tile t = tile;
    t.arr = "tile" + std::to_string(ti++);
    t.b0 = "b0";
    t.a0 = "a0";
    t.swz = true;
    body.line(std::string("__shared__ __align__(16) ") + ctype(en.dtype) + " " + t.arr + "[" + std::to_string(TT * TT) +
              "];");
    em.tiled[e] = t;
  }
  // load phase: thread -> (a-row tid/16 + 16*pass, b-vector tid%16)
  body.line("const int sx_lra = tid >> 4, sx_lb4 = (tid & 15) << 2;");
  for (int pass = 0; pass < TT / 16; ++pass) {
    body.line("{");
    body.indent++;
    em.push();
    const std::string ra = em.fresh("ra"), av = em.fresh("la"), bv = em.fresh("lb");
    body.line("const int " + ra + " = sx_lra + " + std::to_string(16 * pass) + ";");
    body.line("const " + it + " " + av + " = a0 + " + ra + ";");
    body.line("const " + it + " " + bv + " = b0 + sx_lb4;");
    body.line("if (" + av + " < " + fmt_i(na) + " && " + bv + " < " + fmt_i(nb) + ") {");
    body.indent++;
    std::vector<Ix> rc(n);
    rc[a] = em.uni(av);
    rc[b] = em.uni(bv);
    for (size_t k = 0; k < rest_axes.size(); ++k) rc[rest_axes[k]] = rest[k];
    for (auto& [e, tile] : tp.inputs) {
      const Node& en = c.g.nodes[e];
      const Labels& lab = tp.labels.at(e);
      std::vector<Ix> ic(en.rank());
      for (int d = 0; d < en.rank(); ++d) {
        std::string v = "0";
        for (auto& [axis, ext] : lab[d]) v = Emitter::iadd(Emitter::imul(v, ext), rc[axis].e);
        ic[d] = em.uni(em.ivar(v));
      }
      Ix L = em.linearize(ic, en.dims);
      const std::string q = em.fresh("q");
      const char* vt = en.dtype == SFX_F32 ? "sfx_f4" : "sfx_i4";
      body.line(std::string("const ") + vt + " " + q + " = sfx_ld4s(" + em.input_ptr.at(e) + " + " + L.e + ");");
      body.line("*reinterpret_cast<" + std::string(vt) + "*>(&" + em.tiled[e].arr + "[" + ra + " * 64 + (((sx_lb4 >> 2) ^ ((" +
                ra + " >> 2) & 7)) << 2)]) = " + q + ";");
    }
    body.indent--;
    body.line("}");
    em.pop();
    body.indent--;
    body.line("}");
  }
  body.line("__syncthreads();");
  // compute phase: warp w covers a-half (w & 1), b-group (w >> 1); lane l:
  // a-vector l & 7, b offset l >> 3
  body.line("const int sx_cw = tid >> 5, sx_cl = tid & 31;");
  body.line("const int sx_ca4 = ((sx_cw & 1) << 5) + ((sx_cl & 7) << 2), sx_cbo = ((sx_cw >> 1) << 2) + (sx_cl >> 3);");
  for (int pass = 0; pass < TT / 16; ++pass) {
    body.line("{");
    body.indent++;
    em.push();
    const std::string av = em.fresh("ca"), bv = em.fresh("cb");
    body.line("const " + it + " " + av + " = a0 + sx_ca4;");
    body.line("const " + it + " " + bv + " = b0 + sx_cbo + " + std::to_string(16 * pass) + ";");
    body.line("if (" + av + " < " + fmt_i(na) + " && " + bv + " < " + fmt_i(nb) + ") {");
    body.indent++;
    std::vector<std::vector<std::string>> vals(c.p.roots.size(), std::vector<std::string>(4));
    std::string base;
    for (int lane = 0; lane < 4; ++lane) {
      em.lane = lane;
      std::vector<Ix> rc(n);
      rc[a] = em.lane_plus(av);
      rc[b] = em.uni(bv);
      for (size_t k = 0; k < rest_axes.size(); ++k) rc[rest_axes[k]] = rest[k];
      for (size_t r = 0; r < c.p.roots.size(); ++r) vals[r][lane] = em.value(c.p.roots[r], rc);
      if (lane == 0) {
        Ix L = em.linearize(rc, dims);
        if (L.kind != IX_PLUS) throw Error(SFX_ERR_INVALID, "internal: tiled root store is not lane-contiguous");
        base = L.base;
      }
    }
    em.lane = 0;
    for (size_t r = 0; r < c.p.roots.size(); ++r)
      body.line("sfx_st4(out" + std::to_string(root_slot(c, c.p.roots[r])) + " + " + base + ", " + vals[r][0] + ", " +
                vals[r][1] + ", " + vals[r][2] + ", " + vals[r][3] + ");");
    body.indent--;
    body.line("}");
    em.pop();
    body.indent--;
    body.line("}");
  }
  ks.code = assemble(sig, body);
  ks.block = 256;
  ks.grid_x = nta * ntb * nrest;
  ks.vector_width = 4;
  ks.note = "kLoop with " + std::to_string(tp.inputs.size()) + " smem-tiled transposed input(s), tile 64x64 over root "
            "axes (" + std::to_string(a) + "," + std::to_string(b) + "), 128-bit global loads/stores, XOR-swizzled "
            "16-byte chunks";
  return ks;
}

KernelSource lower_map_tiled(const Ctx& c, const TilePlan& tp, const sfx_compile_opts& o) {
  KernelSource ks;
  ks.strategy = "map";
  ks.entry = "sfx_mapt_" + c.name;
  fill_common(c, ks);
  const std::vector<int64_t>& dims = c.g.nodes[c.p.roots[0]].dims;
  const int n = static_cast<int>(dims.size());
  const int a = tp.a, b = tp.b;
  const int64_t na = dims[a], nb = dims[b];
  // TT x TT tiles, 256 threads (32 x 8): 64 keeps 16 loads per thread in
  // flight (32: 4, latency-bound at 4.5 TB/s on C4t); items_per_thread=1
  // selects 32 for A/B
  const int TT = o.items_per_thread == 1 ? 32 : 64;
  // 128-bit path: both tile axes split into 4-vectors, every tiled input's
  // b-run contiguous and 16-byte aligned (its innermost index is b, or b mod a
  // multiple of 4)
  bool vec = TT == 64 && na % 4 == 0 && nb % 4 == 0 && o.row_pipeline != 1;  // row_pipeline=1: scalar tile (A/B)
  for (auto& [e, tile] : tp.inputs) {
    (void)e;
    if (tile.mb != 0 && tile.mb % 4 != 0) vec = false;
  }
  if (vec) return lower_map_tiled_v4(c, tp, o);
  const int64_t nta = (na + TT - 1) / TT, ntb = (nb + TT - 1) / TT;
  std::vector<int64_t> rest_dims;
  std::vector<int> rest_axes;
  for (int i = 0; i < n; ++i)
    if (i != a && i != b) rest_dims.push_back(dims[i]), rest_axes.push_back(i);
  const int64_t nrest = prod(rest_dims, 0, rest_dims.size());
  Emitter em(c.g, c.p, 1, c.wide);
  std::string sig = signature(c, em, ks.entry, 256);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  body.line("const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;");
  body.line(it + " tix = blockIdx.x;");
  body.line("const " + it + " a0 = (tix % " + fmt_i(nta) + ") * " + std::to_string(TT) + "; tix /= " + fmt_i(nta) + ";");
  body.line("const " + it + " b0 = (tix % " + fmt_i(ntb) + ") * " + std::to_string(TT) + "; tix /= " + fmt_i(ntb) + ";");
  body.line("const " + it + " rest = tix;");
  std::vector<Ix> rest = em.from_linear(em.uni("rest"), rest_dims);
  auto root_comps = [&](const std::string& av, const std::string& bv) {
    std::vector<Ix> comps(n);
    comps[a] = em.uni(av);
    comps[b] = em.uni(bv);
    for (size_t k = 0; k < rest_axes.size(); ++k) comps[rest_axes[k]] = rest[k];
    return comps;
  };
  // load phase: each tiled input read along its own innermost dim (root axis b)
  int ti = 0;
  for (auto& [e, tile] : tp.inputs) {
    const Node& en = c.g.nodes[e];
    Emitter::Tile t = tile;
    t.arr = "tile" + std::to_string(ti++);
    t.b0 = "b0";
    t.a0 = "a0";
    body.line(std::string("__shared__ ") + ctype(en.dtype) + " " + t.arr + "[" + std::to_string(TT) + "][" +
              std::to_string(TT + 1) + "];");
    em.tiled[e] = t;
  }
  // input comps for the load phase come from the label walk: rebuild them for
  // (a = a0 + ty + 8k, b = b0 + tx + 32j)
  for (int kj = 0; kj < (TT / 8) * (TT / 32); ++kj) {
    const int k = kj / (TT / 32), j = kj % (TT / 32);
    std::string av = em.fresh("la"), bv = em.fresh("lb");
    body.line("{");
    body.indent++;
    em.push();
    body.line("const " + it + " " + av + " = a0 + ty + " + std::to_string(8 * k) + ";");
    body.line("const " + it + " " + bv + " = b0 + tx + " + std::to_string(32 * j) + ";");
    body.line("if (" + av + " < " + fmt_i(na) + " && " + bv + " < " + fmt_i(nb) + ") {");
    body.indent++;
    std::vector<Ix> rc = root_comps(av, bv);
    for (auto& [e, tile] : tp.inputs) {
      const Node& en = c.g.nodes[e];
      const Labels& lab = tp.labels.at(e);
      std::vector<Ix> ic(en.rank());
      for (int d = 0; d < en.rank(); ++d) {
        std::string v = "0";
        for (auto& [axis, ext] : lab[d]) v = Emitter::iadd(Emitter::imul(v, ext), rc[axis].e);
        ic[d] = em.uni(em.ivar(v));
      }
      Ix L = em.linearize(ic, en.dims);
      body.line(em.tiled[e].arr + "[tx + " + std::to_string(32 * j) + "][ty + " + std::to_string(8 * k) +
                "] = sfx_ld(" + em.input_ptr.at(e) + " + " + L.e + ");");
    }
    body.indent--;
    body.line("}");
    em.pop();
    body.indent--;
    body.line("}");
  }
  body.line("__syncthreads();");
  // compute phase: coalesced along the root's innermost axis a
  for (int kj = 0; kj < (TT / 8) * (TT / 32); ++kj) {
    const int k = kj / (TT / 32), j = kj % (TT / 32);
    std::string av = em.fresh("ca"), bv = em.fresh("cb");
    body.line("{");
    body.indent++;
    em.push();
    body.line("const " + it + " " + av + " = a0 + tx + " + std::to_string(32 * j) + ";");
    body.line("const " + it + " " + bv + " = b0 + ty + " + std::to_string(8 * k) + ";");
    body.line("if (" + av + " < " + fmt_i(na) + " && " + bv + " < " + fmt_i(nb) + ") {");
    body.indent++;
    std::vector<Ix> rc = root_comps(av, bv);
    for (int r : c.p.roots) {
      std::string v = em.value(r, rc);
      Ix L = em.linearize(rc, dims);
      body.line("out" + std::to_string(root_slot(c, r)) + "[" + L.e + "] = " + v + ";");
    }
    body.indent--;
    body.line("}");
    em.pop();
    body.indent--;
    body.line("}");
  }
  ks.code = assemble(sig, body);
  ks.block = 256;
  ks.grid_x = nta * ntb * nrest;
  ks.vector_width = 1;
  ks.note = "kLoop with " + std::to_string(tp.inputs.size()) + " smem-tiled transposed input(s), tile " + std::to_string(TT) + "x" + std::to_string(TT) + " over root axes (" +
            std::to_string(a) + "," + std::to_string(b) + ")";
  return ks;
}

}  // namespace lw
}  // namespace sfx
