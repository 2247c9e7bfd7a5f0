// Group context, kernel scaffolding and the template analyses (GroupAnalyzer).
#include "lower_impl.hpp"

#include <cstdlib>

namespace sfx {
namespace lw {

enum { CLS_NONE = 0, CLS_FULL = 1, CLS_ROWV = 2, CLS_COLV = 3 };


int64_t prod(const std::vector<int64_t>& d, size_t b, size_t e) {
  int64_t n = 1;
  for (size_t i = b; i < e; ++i) n *= d[i];
  return n;
}

std::string sanitize(const std::string& s) {
  std::string o;
  for (char c : s) o += (std::isalnum(static_cast<unsigned char>(c)) ? c : '_');
  if (o.size() > 40) o.resize(40);
  return o;
}

// A reduction over extent-1 dims folds one element: the element itself (the
// reference's fold starts from the first element, exec.cpp:196-201), i.e. a
// reshape.  Such reduces are index algebra, not reductions, for the analyzers.
bool degenerate_reduce(const Graph& g, const Node& n) {
  return n.op == SFX_OP_REDUCE && g.nodes[n.operands[0]].numel() == n.numel();
}

Ctx make_ctx(const Graph& g, const Program& p) {
  Ctx c(g, p);
  std::set<int> seen;
  std::function<void(int)> visit = [&](int n) {
    if (!p.is_member(n) || seen.count(n)) return;
    seen.insert(n);
    for (int op : g.nodes[n].operands) visit(op);
    c.topo.push_back(n);
  };
  for (int m : p.members) visit(m);
  for (int m : c.topo) {
    const Node& n = g.nodes[m];
    if (n.op == SFX_OP_LIBRARY_CALL)  // always a fusion barrier (span.cpp:35)
      throw Error(SFX_ERR_INVALID, "group member " + n.id + " is a library call");
    if (n.op == SFX_OP_BATCH_MATMUL) c.dots.push_back(m);
    const bool real_reduce = n.op == SFX_OP_REDUCE && !degenerate_reduce(g, n);
    bool d = real_reduce;
    for (int op : n.operands)
      if (p.is_member(op) && c.dep[op]) d = true;
    c.dep[m] = d;
    if (real_reduce) c.reduces.push_back(m);
  }
  int64_t big = 0;
  for (int m : p.members) big = std::max(big, g.nodes[m].numel());
  for (int e : p.externals) big = std::max(big, g.nodes[e].numel());
  c.wide = big >= (int64_t{1} << 30) || p.blocks >= (int64_t{1} << 30);
  c.name = sanitize(g.nodes[p.fusion_root >= 0 ? p.fusion_root : p.roots[0]].id);
  return c;
}

bool rcp_divisors() {
  const char* e = std::getenv("SFX_EXACT_DIV");
  return !(e && e[0] == '1');
}

// External f32 inputs with `full` elements that the group reads only at the
// element being computed (every path from a root or a reduction's operand goes
// through linear-index-preserving edges: elementwise, reshape / bitcast,
// reshape-like broadcast / transpose, degenerate reduce) — safe to stage per
// thread in shared memory at the thread's own element.
std::set<int> identity_inputs(const Ctx& c, int64_t full) {
  const Graph& g = c.g;
  std::set<int> local, unsafe;
  std::set<std::pair<int, bool>> seen;
  std::function<void(int, bool)> walk = [&](int n, bool ok) {
    if (!seen.insert({n, ok}).second) return;
    const Node& m = g.nodes[n];
    if (!c.p.is_member(n)) {
      if (m.numel() == full) (ok ? local : unsafe).insert(n);
      return;
    }
    if (m.op == SFX_OP_REDUCE && !degenerate_reduce(g, m)) {
      for (int o : m.operands) walk(o, g.nodes[o].numel() == full);
      return;
    }
    bool edge = false;
    if (m.numel() == full) switch (m.op) {
        case SFX_OP_ELEMENTWISE: case SFX_OP_RESHAPE: case SFX_OP_BITCAST: case SFX_OP_REDUCE:
          edge = true;
          break;
        case SFX_OP_BROADCAST:
          edge = bcast_is_reshape(m);
          break;
        case SFX_OP_TRANSPOSE:
          edge = transpose_is_reshape(m);
          break;
        default:
          break;
      }
    for (int o : m.operands) walk(o, ok && edge);
  };
  for (int r : c.p.roots) walk(r, g.nodes[r].numel() == full);
  std::set<int> out;
  for (int e : local)
    if (!unsafe.count(e) && g.nodes[e].dtype == SFX_F32) out.insert(e);
  return out;
}

// ---- kernel scaffolding ---------------------------------------------------

std::string signature(const Ctx& c, Emitter& em, const std::string& entry, int block, int min_blocks,
                      bool stream) {
  std::ostringstream os;
  os << "extern \"C\" __global__ void __launch_bounds__(" << block;
  if (min_blocks > 0) os << ", " << min_blocks;
  os << ") " << entry << "(";
  bool first = true;
  for (size_t k = 0; k < c.p.inputs.size(); ++k) {
    int n = c.p.inputs[k];
    std::string name = "in" + std::to_string(k);
    os << (first ? "" : ", ") << "const " << ctype(c.g.nodes[n].dtype) << "* __restrict__ " << name;
    first = false;
    em.input_ptr[n] = name;
    if (c.g.nodes[n].numel() * 4 >= (int64_t{1} << 20)) em.streaming.insert(n);
  }
  for (size_t r = 0; r < c.p.roots.size(); ++r) {
    os << (first ? "" : ", ") << ctype(c.g.nodes[c.p.roots[r]].dtype) << "* __restrict__ out" << r;
    first = false;
  }
  os << (first ? "" : ", ") << "unsigned* __restrict__ ws";
  if (c.peer)
    os << ", const unsigned long long* __restrict__ peers, unsigned long long poff, int prank, int pn";
  if (stream) os << ", const unsigned* __restrict__ sgate, unsigned* __restrict__ sdone, long long schunk";
  os << ")";
  return os.str();
}

void fill_common(const Ctx& c, KernelSource& ks) {
  ks.inputs = c.p.inputs;
  ks.outputs = c.p.roots;
  int64_t b = 0;
  for (int n : c.p.inputs) b += c.g.nodes[n].numel() * 4;
  for (int n : c.p.roots) b += c.g.nodes[n].numel() * 4;
  ks.algorithmic_bytes = b;
}

std::string assemble(const std::string& sig, const Code& body) {
  std::string s;
  if (const char* e = std::getenv("SFX_EXPERIMENT"))  // A/B experiments only (tools/)
    s += std::string("#define ") + e + " 1\n";
  s += kPrelude;
  s += "\n";
  s += sig;
  s += " {\n";
  // Programmatic dependent launch: the runtime launches this grid while the
  // previous one drains; wait here until that grid's writes are visible
  // (full dependency kept), then let the next grid launch early.
  s += "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  s += "  asm volatile(\"griddepcontrol.launch_dependents;\" :::);\n";
  s += body.text;
  s += "}\n";
  return s;
}

// Host-streaming gate (see KernelSource::stream_R): emitted first in the body.
// `e0` = the CTA's first element of the [R, C] row space; a CTA never spans
// two chunks, so it waits for its own chunk's copies (a copy stream sets
// sgate[j] = 1 after chunk j).
void emit_stream_gate(Code& body, const std::string& e0, int64_t cta_elems, int64_t total) {
  // all of it behind the (uniform) null test: the device path pays one branch
  body.line("if (sgate) {");
  body.line("  const long long s_e1 = min(" + e0 + " + (long long)" + fmt_i(cta_elems) + ", (long long)" +
            fmt_i(total) + ") - 1;");
  body.line("  if (threadIdx.x == 0) sfx_gate_wait(sgate + s_e1 / schunk, 1u);");
  body.line("  __syncthreads();");
  body.line("}");
}
// ... and last: once every thread's stores are issued, one release-ordered
// increment of the chunk's completion counter (the copy-back stream waits for
// the chunk's CTA count with cuStreamWaitValue32).
void emit_stream_done(Code& body, const std::string& e0) {
  body.line("if (sdone) {");
  body.line("  __syncthreads();");
  body.line("  if (threadIdx.x == 0) { __threadfence(); atomicAdd(sdone + (" + e0 + ") / schunk, 1u); }");
  body.line("}");
}

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

int root_slot(const Ctx& c, int node) {
  for (size_t r = 0; r < c.p.roots.size(); ++r)
    if (c.p.roots[r] == node) return static_cast<int>(r);
  return -1;
}

// index component splitting a linear (row, col) pair for a node of `dims`,
// when its dims split as [row dims | col dims] with prod(row dims) == R
int prefix_split(const std::vector<int64_t>& dims, int64_t R) {
  int64_t acc = 1;
  for (size_t k = 0; k <= dims.size(); ++k) {
    if (acc == R) return static_cast<int>(k);
    if (k < dims.size()) acc *= dims[k];
  }
  return -1;
}

std::vector<Ix> rowcol_comps(Emitter& em, const std::vector<int64_t>& dims, int64_t R, int64_t C,
                             const Ix& row, const Ix& col) {
  int k = prefix_split(dims, R);
  if (k >= 0 && prod(dims, k, dims.size()) == C) {
    std::vector<int64_t> rd(dims.begin(), dims.begin() + k), cd(dims.begin() + k, dims.end());
    std::vector<Ix> a = em.from_linear(row, rd);
    std::vector<Ix> b = em.from_linear(col, cd);
    a.insert(a.end(), b.begin(), b.end());
    return a;
  }
  // no [row|col] split of this shape: go through the linear index
  Ix L;
  std::string rb = em.ivar(Emitter::imul(row.e, C));
  if (col.kind == IX_PLUS) {
    L = em.lane_plus(em.ivar(Emitter::iadd(rb, col.base)));
  } else {
    L = em.uni(em.ivar(Emitter::iadd(rb, col.e)));
    L.kind = col.kind;
  }
  return em.from_linear(L, dims);
}

bool bcast_is_reshape(const Node& m) {
  std::set<int64_t> mapped(m.dim_map.begin(), m.dim_map.end());
  for (int i = 0; i < m.rank(); ++i)
    if (!mapped.count(i) && m.dims[i] != 1) return false;
  return true;
}

bool transpose_is_reshape(const Node& m) {
  int64_t prev = -1;
  for (int i = 0; i < m.rank(); ++i) {
    if (m.dims[i] == 1) continue;
    if (m.perm[i] < prev) return false;
    prev = m.perm[i];
  }
  return true;
}

// ---- ROW analysis ------------------------------------------------------------


bool analyze_row(const Ctx& c, RowPlan* rp, std::string* why) {
  const Graph& g = c.g;
  if (!c.dots.empty()) return *why = "group contains a matmul", false;
  if (c.reduces.empty()) return *why = "no reduction", false;
  for (int r : c.reduces) {
    const Node& n = g.nodes[r];
    const Node& in = g.nodes[n.operands[0]];
    std::vector<int64_t> rd = n.reduce_dims;
    std::sort(rd.begin(), rd.end());
    int k = in.rank() - static_cast<int>(rd.size());
    for (size_t i = 0; i < rd.size(); ++i)
      if (rd[i] != k + static_cast<int64_t>(i)) return *why = "reduce " + n.id + " is not over trailing dims", false;
    int64_t R = prod(in.dims, 0, k), C = prod(in.dims, k, in.dims.size());
    if (rp->R == 0) {
      rp->R = R;
      rp->C = C;
    } else if (rp->R != R || rp->C != C) {
      return *why = "reductions with different row geometry", false;
    }
  }
  if (rp->C <= 1) return *why = "degenerate row length", false;
  const int64_t R = rp->R, C = rp->C;
  auto cls_of_numel = [&](int64_t n) { return n == R * C ? CLS_FULL : (n == R ? CLS_ROWV : CLS_NONE); };
  for (int m : c.topo) {
    const Node& n = g.nodes[m];
    if (!c.dep.at(m)) continue;
    int cls = cls_of_numel(n.numel());
    if (n.op == SFX_OP_REDUCE && !degenerate_reduce(g, n)) {
      int op = n.operands[0];
      if (c.p.is_member(op) && c.dep.at(op) && rp->cls[op] != CLS_FULL)
        return *why = "reduce operand " + g.nodes[op].id + " is not row-shaped", false;
      rp->cls[m] = CLS_ROWV;
      int lv = 1;
      std::function<void(int)> walk;
      std::set<int> seen;
      walk = [&](int x) {
        if (!c.p.is_member(x) || seen.count(x)) return;
        seen.insert(x);
        if (x != m && g.nodes[x].op == SFX_OP_REDUCE) lv = std::max(lv, rp->level[x] + 1);
        if (x == m || g.nodes[x].op != SFX_OP_REDUCE)
          for (int o : g.nodes[x].operands) walk(o);
      };
      walk(m);
      rp->level[m] = lv;
      rp->max_level = std::max(rp->max_level, lv);
      continue;
    }
    if (cls == CLS_NONE) return *why = "member " + n.id + " is neither row- nor element-shaped", false;
    for (int op : n.operands) {
      if (!c.p.is_member(op) || !c.dep.at(op)) continue;
      int oc = rp->cls[op];
      const Node& o = g.nodes[op];
      switch (n.op) {
        case SFX_OP_ELEMENTWISE:
        case SFX_OP_RESHAPE:
        case SFX_OP_BITCAST:
        case SFX_OP_REDUCE:  // degenerate: a reshape
          if (oc != cls) return *why = "class mismatch at " + n.id, false;
          break;
        case SFX_OP_BROADCAST: {
          if (bcast_is_reshape(n) && oc == cls) break;
          bool prefix = cls == CLS_FULL && oc == CLS_ROWV;
          for (size_t j = 0; prefix && j < n.dim_map.size(); ++j)
            if (n.dim_map[j] != static_cast<int64_t>(j)) prefix = false;
          if (prefix && prod(n.dims, n.dim_map.size(), n.dims.size()) == C) break;
          return *why = "broadcast " + n.id + " does not map rows to rows", false;
        }
        case SFX_OP_TRANSPOSE: {
          if (oc != cls) return *why = "class mismatch at " + n.id, false;
          if (transpose_is_reshape(n)) break;
          int k = prefix_split(n.dims, R);
          bool ok = cls == CLS_FULL && k >= 0;
          for (int i = 0; ok && i < k; ++i)
            if (n.perm[i] != i) ok = false;
          if (ok) break;
          return *why = "transpose " + n.id + " moves data across rows", false;
        }
        default:
          return *why = "unsupported op at " + n.id, false;
      }
      (void)o;
    }
    rp->cls[m] = cls;
  }
  for (int r : c.p.roots) {
    int cls = cls_of_numel(g.nodes[r].numel());
    if (cls == CLS_NONE) return *why = "root " + g.nodes[r].id + " is neither row- nor element-shaped", false;
    if (c.dep.at(r) && rp->cls[r] != cls) return *why = "root class mismatch", false;
  }
  return true;
}

// ---- COL analysis ------------------------------------------------------------


bool analyze_col(const Ctx& c, ColPlan* cp, std::string* why) {
  const Graph& g = c.g;
  if (!c.dots.empty()) return *why = "group contains a matmul", false;
  if (c.reduces.empty()) return *why = "no reduction", false;
  for (int r : c.reduces) {
    const Node& n = g.nodes[r];
    const Node& in = g.nodes[n.operands[0]];
    if (c.p.is_member(n.operands[0]) && c.dep.at(n.operands[0]))
      return *why = "nested reduction at " + n.id, false;
    std::vector<int64_t> rd = n.reduce_dims;
    std::sort(rd.begin(), rd.end());
    for (size_t i = 0; i < rd.size(); ++i)
      if (rd[i] != rd[0] + static_cast<int64_t>(i)) return *why = "reduce " + n.id + " dims are not contiguous", false;
    const int k0 = static_cast<int>(rd[0]), k1 = static_cast<int>(rd.back()) + 1;
    int64_t O = prod(in.dims, 0, k0), R = prod(in.dims, k0, k1), I = prod(in.dims, k1, in.dims.size());
    if (cp->R == 0) {
      cp->O = O;
      cp->R = R;
      cp->I = I;
    } else if (cp->O != O || cp->R != R || cp->I != I) {
      return *why = "column reductions with different geometry", false;
    }
  }
  const int64_t R = cp->R, C = cp->O * cp->I;
  if (R <= 1) return *why = "degenerate column length", false;
  for (int m : c.topo) {
    const Node& n = g.nodes[m];
    if (!c.dep.at(m) || n.op == SFX_OP_REDUCE) continue;
    if (n.numel() != C) return *why = "member " + n.id + " needs the reduced columns broadcast back", false;
    switch (n.op) {
      case SFX_OP_ELEMENTWISE:
      case SFX_OP_RESHAPE:
      case SFX_OP_BITCAST:
        break;
      case SFX_OP_BROADCAST:
        if (!bcast_is_reshape(n)) return *why = "broadcast of reduced columns at " + n.id, false;
        break;
      case SFX_OP_TRANSPOSE:
        if (!transpose_is_reshape(n)) return *why = "transpose of reduced columns at " + n.id, false;
        break;
      default:
        return *why = "unsupported op at " + n.id, false;
    }
  }
  for (int r : c.p.roots) {
    int64_t n = g.nodes[r].numel();
    if (c.dep.at(r)) {
      if (n != C) return *why = "root " + g.nodes[r].id + " mixes reduced and unreduced data", false;
    } else if (n != R * C && n != C) {
      return *why = "root " + g.nodes[r].id + " has unrelated shape", false;
    }
  }
  return true;
}

// ---- COL with broadcast-back analysis (batch-norm statistics) ------------------


bool analyze_colbc(const Ctx& c, ColBcPlan* bp, std::string* why) {
  const Graph& g = c.g;
  if (!c.dots.empty()) return *why = "group contains a matmul", false;
  if (c.reduces.empty()) return *why = "no reduction", false;
  std::vector<int> kept;  // FULL-space axes that survive the reductions (of the reduce operands)
  for (int r : c.reduces) {
    const Node& n = g.nodes[r];
    const Node& in = g.nodes[n.operands[0]];
    std::vector<int64_t> rd = n.reduce_dims;
    std::sort(rd.begin(), rd.end());
    for (size_t i = 0; i < rd.size(); ++i)
      if (rd[i] != rd[0] + static_cast<int64_t>(i)) return *why = "reduce " + n.id + " dims are not contiguous", false;
    const int k0 = static_cast<int>(rd[0]), k1 = static_cast<int>(rd.back()) + 1;
    const int64_t O = prod(in.dims, 0, k0), R = prod(in.dims, k0, k1), I = prod(in.dims, k1, in.dims.size());
    if (bp->R == 0) {
      bp->O = O, bp->R = R, bp->I = I;
    } else if (bp->O != O || bp->R != R || bp->I != I) {
      return *why = "column reductions with different geometry", false;
    }
  }
  const int64_t O = bp->O, R = bp->R, I = bp->I, C = O * I;
  if (R <= 1) return *why = "degenerate column length", false;
  enum { FULL = 1, COLV = 2 };
  std::map<int, int> cls;
  auto cls_of = [&](int64_t n) { return n == O * R * I ? FULL : n == C ? COLV : 0; };
  for (int m : c.topo) {
    const Node& n = g.nodes[m];
    if (!c.dep.at(m)) continue;
    if (n.op == SFX_OP_REDUCE && !degenerate_reduce(g, n)) {
      int op = n.operands[0];
      if (c.p.is_member(op) && c.dep.at(op) && cls[op] != FULL)
        return *why = "reduce operand " + g.nodes[op].id + " is not element-shaped", false;
      cls[m] = COLV;
      int lv = 1;
      std::set<int> seen;
      std::function<void(int)> walk = [&](int x) {
        if (!c.p.is_member(x) || seen.count(x)) return;
        seen.insert(x);
        if (x != m && g.nodes[x].op == SFX_OP_REDUCE && !degenerate_reduce(g, g.nodes[x]))
          lv = std::max(lv, bp->level[x] + 1);
        else
          for (int o : g.nodes[x].operands) walk(o);
      };
      for (int o : n.operands) walk(o);
      bp->level[m] = lv;
      bp->max_level = std::max(bp->max_level, lv);
      continue;
    }
    int k = cls_of(n.numel());
    if (!k) return *why = "member " + n.id + " is neither element- nor column-shaped", false;
    for (int op : n.operands) {
      if (!c.p.is_member(op) || !c.dep.at(op)) continue;
      int oc = cls[op];
      switch (n.op) {
        case SFX_OP_ELEMENTWISE:
        case SFX_OP_RESHAPE:
        case SFX_OP_BITCAST:
        case SFX_OP_REDUCE:  // degenerate
          if (oc != k) return *why = "class mismatch at " + n.id, false;
          break;
        case SFX_OP_TRANSPOSE:
          if (oc != k || !transpose_is_reshape(n)) return *why = "transpose of dependent data at " + n.id, false;
          break;
        case SFX_OP_BROADCAST: {
          if (bcast_is_reshape(n) && oc == k) break;
          // columns broadcast back over the reduced block: the output splits as
          // [O dims | R dims | I dims] and the operand maps onto the O and I dims
          int k0 = prefix_split(n.dims, O), k1 = k0 < 0 ? -1 : prefix_split(n.dims, O * R);
          bool ok = k == FULL && oc == COLV && k0 >= 0 && k1 >= k0 && prod(n.dims, k1, n.dims.size()) == I;
          std::vector<int64_t> want;
          for (int d = 0; d < n.rank(); ++d)
            if ((d < k0 || d >= k1) && n.dims[d] != 1) want.push_back(d);
          std::vector<int64_t> have;
          for (size_t j = 0; j < n.dim_map.size(); ++j)
            if (g.nodes[op].dims[j] != 1) have.push_back(n.dim_map[j]);
          if (!ok || want != have) return *why = "broadcast " + n.id + " does not map columns to columns", false;
          break;
        }
        default:
          return *why = "unsupported op at " + n.id, false;
      }
    }
    cls[m] = k;
  }
  bool back = false;  // at least one reduction feeds an element again
  for (int m : c.topo)
    if (c.dep.at(m) && cls[m] == FULL) back = true;
  if (!back) return *why = "no broadcast back (column template)", false;
  for (int r : c.p.roots) {
    int k = cls_of(c.g.nodes[r].numel());
    if (!k) return *why = "root " + g.nodes[r].id + " is neither element- nor column-shaped", false;
    if (c.dep.at(r) && cls[r] != k) return *why = "root class mismatch", false;
  }
  return true;
}

bool analyze_colbc_split(const Ctx& c, SplitPlan* sp, std::string* why) {
  const Graph& g = c.g;
  if (!c.dots.empty()) return *why = "group contains a matmul", false;
  if (c.reduces.empty()) return *why = "no reduction", false;
  for (int r : c.reduces) {
    const Node& n = g.nodes[r];
    const Node& in = g.nodes[n.operands[0]];
    if (n.reducer != SFX_REDUCE_SUM || n.dtype != SFX_F32) return *why = "reduce " + n.id + " is not an f32 sum", false;
    std::vector<bool> red(in.rank(), false);
    for (int64_t d : n.reduce_dims) red[d] = true;
    int k0 = 0;
    while (k0 < in.rank() && red[k0]) ++k0;
    int k1 = k0;
    while (k1 < in.rank() && !red[k1]) ++k1;
    for (int d = k1; d < in.rank(); ++d)
      if (!red[d]) return *why = "reduce " + n.id + " keeps a non-contiguous dim block", false;
    if (k0 == 0 || k1 == in.rank()) return *why = "reduce " + n.id + " dims are contiguous (colbc)", false;
    const int64_t A = prod(in.dims, 0, k0), K = prod(in.dims, k0, k1), B = prod(in.dims, k1, in.dims.size());
    if (sp->K == 0) {
      sp->A = A, sp->K = K, sp->B = B;
    } else if (sp->A != A || sp->K != K || sp->B != B) {
      return *why = "reductions with different geometry", false;
    }
  }
  const int64_t A = sp->A, K = sp->K, B = sp->B;
  if (A * B <= 1 || K == A * K * B) return *why = "degenerate channel length", false;
  enum { FULL = 1, CHAN = 2 };
  std::map<int, int> cls;
  auto cls_of = [&](int64_t n) { return n == A * K * B ? FULL : n == K ? CHAN : 0; };
  for (int m : c.topo) {
    const Node& n = g.nodes[m];
    if (!c.dep.at(m)) continue;
    if (n.op == SFX_OP_REDUCE && !degenerate_reduce(g, n)) {
      int op = n.operands[0];
      if (c.p.is_member(op) && c.dep.at(op) && cls[op] != FULL)
        return *why = "reduce operand " + g.nodes[op].id + " is not element-shaped", false;
      cls[m] = CHAN;
      int lv = 1;
      std::set<int> seen;
      std::function<void(int)> walk = [&](int x) {
        if (!c.p.is_member(x) || seen.count(x)) return;
        seen.insert(x);
        if (x != m && g.nodes[x].op == SFX_OP_REDUCE && !degenerate_reduce(g, g.nodes[x]))
          lv = std::max(lv, sp->level[x] + 1);
        else
          for (int o : g.nodes[x].operands) walk(o);
      };
      for (int o : n.operands) walk(o);
      sp->level[m] = lv;
      sp->max_level = std::max(sp->max_level, lv);
      continue;
    }
    int k = cls_of(n.numel());
    if (!k) return *why = "member " + n.id + " is neither element- nor channel-shaped", false;
    for (int op : n.operands) {
      if (!c.p.is_member(op) || !c.dep.at(op)) continue;
      int oc = cls[op];
      switch (n.op) {
        case SFX_OP_ELEMENTWISE:
        case SFX_OP_RESHAPE:
        case SFX_OP_BITCAST:
        case SFX_OP_REDUCE:  // degenerate
          if (oc != k) return *why = "class mismatch at " + n.id, false;
          break;
        case SFX_OP_TRANSPOSE:
          if (oc != k || !transpose_is_reshape(n)) return *why = "transpose of dependent data at " + n.id, false;
          break;
        case SFX_OP_BROADCAST: {
          if (bcast_is_reshape(n) && oc == k) break;
          // channels broadcast back: the output splits as [A dims | K dims | B dims]
          // and the operand maps onto the K dims
          int k0 = prefix_split(n.dims, A), k1 = k0 < 0 ? -1 : prefix_split(n.dims, A * K);
          bool ok = k == FULL && oc == CHAN && k0 >= 0 && k1 >= k0 && prod(n.dims, k1, n.dims.size()) == B;
          std::vector<int64_t> want;
          for (int d = 0; d < n.rank(); ++d)
            if (d >= k0 && d < k1 && n.dims[d] != 1) want.push_back(d);
          std::vector<int64_t> have;
          for (size_t j = 0; j < n.dim_map.size(); ++j)
            if (g.nodes[op].dims[j] != 1) have.push_back(n.dim_map[j]);
          if (!ok || want != have) return *why = "broadcast " + n.id + " does not map channels to channels", false;
          break;
        }
        default:
          return *why = "unsupported op at " + n.id, false;
      }
    }
    cls[m] = k;
  }
  for (int r : c.p.roots) {
    int k = cls_of(c.g.nodes[r].numel());
    if (!k) return *why = "root " + g.nodes[r].id + " is neither element- nor channel-shaped", false;
    if (c.dep.at(r) && cls[r] != k) return *why = "root class mismatch", false;
  }
  return true;
}

}  // namespace lw
}  // namespace sfx
