#include "lower.hpp"

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

namespace {

constexpr int kNumSMs = 148;

enum { CLS_NONE = 0, CLS_FULL = 1, CLS_ROWV = 2, CLS_COLV = 3 };

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

// ---- kernel scaffolding ---------------------------------------------------

std::string signature(const Ctx& c, Emitter& em, const std::string& entry, int block, int min_blocks = 0,
                      bool stream = false) {
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

struct RowPlan {
  int64_t R = 0, C = 0;
  std::map<int, int> cls;
  std::map<int, int> level;
  int max_level = 0;
};

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

struct ColPlan {
  int64_t O = 0, R = 0, I = 0;  // [outer | reduced | inner] of every reduce operand
};

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
constexpr int kUnknown = -2;
using DimLabel = std::vector<std::pair<int, int64_t>>;
using Labels = std::vector<DimLabel>;

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

struct TilePlan {
  int a = -1, b = -1;  // root axes: a = innermost (output-coalesced), b = input-innermost
  std::map<int, Emitter::Tile> inputs;  // external -> where axes a and b sit in its index
  std::map<int, Labels> labels;         // external -> its labelling
};

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

// ---- ROW ------------------------------------------------------------------------

void emit_row_body(const Ctx& c, const RowPlan& rp, Emitter& em, Code& body, int TPR, int V, int64_t NCH);

// Threads per row: the largest power of two <= 32 dividing the row into
// V-vectors; rows longer than 32 threads x 32 elements span several warps (up
// to a whole CTA) at ~32 elements per thread.
// `streams` = number of [R, C] inputs read per element: rows are widened until
// a thread holds <= 32 streamed values (measured on B200: BERT probs_d / h1
// with 3 streamed inputs gain 4-6% at 2 warps per row; 1-input softmax rows
// are best at one warp).
int row_tpr(int64_t C, int V, int streams = 1) {
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
KernelSource lower_row_mp(const Ctx& c, const RowPlan& rp, const sfx_compile_opts& o) {
  KernelSource ks;
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
    const int cs_max = o.pipe_stages == 16 ? 16 : 8;
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
  if (CS > 1 && persist) {
    body.line("const unsigned q = sfx_cluster_rank();");
    body.line("const " + it + " cid = (" + it + ")blockIdx.x / " + std::to_string(CS) + ";");
    body.line("extern __shared__ __align__(128) unsigned char sfx_smem[];");
    body.line("unsigned long long* sbar = (unsigned long long*)(sfx_smem + " + fmt_i(2 * stage_bytes) + ");");
    body.line("if (tid == 0) {");
    body.line("  sfx_mbar_init(sbar, 1);");
    body.line("  sfx_mbar_init(sbar + 1, 1);");
    body.line("  sfx_fence_mbar_init();");
    body.line("  if (cid < " + fmt_i(R) + ") {");
    issue("0", "cid", "sbar");
    body.line("  }");
    body.line("  if (cid + " + fmt_i(NCL) + " < " + fmt_i(R) + ") {");
    issue("1", "cid + " + fmt_i(NCL), "sbar + 1");
    body.line("  }");
    body.line("}");
    body.line("__syncthreads();");
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
    body.line("  sfx_fence_mbar_init();");
    body.line("  sfx_mbar_expect_tx(sbar, " + fmt_i(bar_off) + "u);");
    for (size_t k = 0; k < staged.size(); ++k)
      body.line("  sfx_bulk_g2s(sfx_smem + " + fmt_i(static_cast<int64_t>(k) * slice_bytes) + ", " +
                em.input_ptr.at(staged[k]) + " + row * " + fmt_i(C) + " + (" + it + ")q * " + fmt_i(SL) + ", " +
                fmt_i(slice_bytes) + "u, sbar);");
    body.line("}");
    body.line("__syncthreads();");
    body.line("sfx_mbar_wait(sbar, 0);");
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
          const Node& rn = c.g.nodes[red[k]];
          const Node& in = c.g.nodes[rn.operands[0]];
          std::string v = em.value(rn.operands[0], rowcol_comps(em, in.dims, R, C, rowix, col));
          body.line(acc[k] + " = " + fold_of(rn) + "(" + acc[k] + ", " + v + ");");
        }
      }
    });
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
      if (CS > 1) {
        // cluster combine: every CTA folds the CS partials in rank order
        const std::string xp = em.fresh("xp");
        body.line("__shared__ " + T + " " + xp + ";");
        body.line("if (tid == 0) " + xp + " = " + acc[k] + ";");
        body.line("sfx_cluster_sync();");
        body.line(acc[k] + " = sfx_dsmem_ld(&" + xp + ", 0u);");
        body.line("for (unsigned r = 1; r < " + std::to_string(CS) + "u; ++r) " + acc[k] + " = " + fold_of(rn) + "(" +
                  acc[k] + ", sfx_dsmem_ld(&" + xp + ", r));");
      }
      std::string fin = acc[k];
      if (T == "double") {
        fin = em.fresh("red");
        body.line("const float " + fin + " = (float)" + acc[k] + ";");
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
  if (CS > 1) body.line("sfx_cluster_sync();  // no CTA leaves while a peer may still read its partials");
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
              " input slice(s) of " + std::to_string(slice_bytes) + " B in shared memory (TMA), DSMEM combine, levels=" +
              std::to_string(rp.max_level) + (persist ? ", persistent: " + std::to_string(NCL) + " clusters, 2 stages" : "");
  else
    ks.note = "rows=" + std::to_string(R) + " cols=" + std::to_string(C) + " one CTA of " + std::to_string(B) +
              " threads per row, multi-pass (" + std::to_string(rp.max_level + (full_roots.empty() ? 0 : 1)) +
              " passes, re-reads from L2) levels=" + std::to_string(rp.max_level);
  return ks;
}

// The row body shared by the register-resident and the TMA-pipelined row
// templates: reduction phases (per-thread fold -> shuffle tree -> broadcast
// back through registers) then the element and row roots.  Expects `row`,
// `lr` (lane within the row group), `gmask`, `gleader` in scope.
void emit_row_body(const Ctx& c, const RowPlan& rp, Emitter& em, Code& body, int TPR, int V, int64_t NCH) {
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

  for (int lv = 1; lv <= rp.max_level; ++lv) {
    std::vector<int> red;
    for (int r : c.reduces)
      if (rp.level.at(r) == lv) red.push_back(r);
    std::vector<std::string> acc(red.size()), first(red.size());
    for (size_t k = 0; k < red.size(); ++k) {
      acc[k] = em.fresh("acc");
      body.line(std::string(ctype(c.g.nodes[red[k]].dtype)) + " " + acc[k] + ";");
    }
    for (int64_t j = 0; j < NCH; ++j)
      for (int lane = 0; lane < V; ++lane) {
        Ix col = col_ix(j, lane);
        for (size_t k = 0; k < red.size(); ++k) {
          const Node& rn = c.g.nodes[red[k]];
          const Node& in = c.g.nodes[rn.operands[0]];
          std::vector<Ix> comps = rowcol_comps(em, in.dims, R, C, rowix, col);
          std::string v = em.value(rn.operands[0], comps);
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
        body.line(acc[k] + " = " + f + "(" + acc[k] + ", sfx_shfl_xor(" + acc[k] + ", " +
                  std::to_string(m) + ", gmask));");
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
        body.line(std::string("__shared__ ") + ctype(rn.dtype) + " " + rsm[k] + "[" + std::to_string(RPC) + "][" +
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
    for (size_t k = 0; k < red.size(); ++k) {
      const Node& rn = c.g.nodes[red[k]];
      if (rn.reducer != SFX_REDUCE_SUM && rn.dtype == SFX_F32) {
        std::string f0 = W > 1 ? rfm[k] + "[rin]" : TPR > 1 ? "sfx_shfl(" + first[k] + ", gleader, gmask)" : first[k];
        body.line(acc[k] + " = sfx_fold_first(" + f0 + ", " + acc[k] + ");");
      }
      reduced[red[k]] = acc[k];
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
  const int UR = o.items_per_thread > 0 ? std::min(o.items_per_thread, 16) : 8;
  const int NR = static_cast<int>(c.reduces.size());
  Emitter em(c.g, c.p, V, c.wide);
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
  // flight together), then the remainder
  auto stripe_pass = [&](const std::function<void(const std::string&)>& row) {
    body.line("if (cok) {");
    body.indent++;
    const std::string r = em.fresh("r");
    body.line(it + " " + r + " = r_begin + rsub;");
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
  for (int lv = 1; lv <= bp.max_level; ++lv) {
    std::vector<int> red;
    for (int r : c.reduces)
      if (bp.level.at(r) == lv) red.push_back(r);
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
          const Node& rn = c.g.nodes[red[k]];
          const Node& in = c.g.nodes[rn.operands[0]];
          std::string v = em.value(rn.operands[0], orc_comps(em, in.dims, O, R, I, oix, rix, iix));
          body.line(acc[k][l] + " = " + fold_fn(red[k]) + "(" + acc[k][l] + ", " + v + ");");
        }
      }
    });
    // CTA combine over row sub-streams (deterministic order), partials out
    for (size_t k = 0; k < red.size(); ++k) {
      const std::string T = acc_t(red[k]);
      const std::string sp = em.fresh("sp");
      body.line("__shared__ " + T + " " + sp + "[" + std::to_string(RSUB) + "][" + fmt_i(TC) + "];");
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
    for (size_t k = 0; k < red.size(); ++k) {
      const Node& rn = c.g.nodes[red[k]];
      const std::string T = acc_t(red[k]);
      std::vector<std::string> tv(V);
      for (int l = 0; l < V; ++l) {
        tv[l] = em.fresh("tot");
        body.line(T + " " + tv[l] + " = __ldcg((const " + T + "*)((const unsigned long long*)(ws + " +
                  fmt_i(tot_word[red[k]]) + ") + (cok ? c0 : 0) + " + std::to_string(l) + "));");
      }
      if (c.peer) {  // the ranks' totals, in rank order (identical on every rank)
        body.line("if (pn > 1) {");
        body.line("  const long long par = (launch_seq * " + std::to_string(bp.max_level) + "u + " + std::to_string(lv) +
                  "u) & 1u;");
        body.line("  const unsigned long long* xs = (const unsigned long long*)(peers[prank] + poff) + (par * " +
                  std::to_string(PMAX) + " * " + std::to_string(NR) + " + " + std::to_string(red_index[red[k]]) + ") * " +
                  fmt_i(C) + " + (cok ? c0 : 0);");
        for (int l = 0; l < V; ++l) {
          body.line("  " + tv[l] + " = __ldcv((const " + T + "*)(xs + " + std::to_string(l) + "));");
          body.line("  for (int q = 1; q < pn; ++q) " + tv[l] + " = " + fold_fn(red[k]) + "(" + tv[l] + ", __ldcv((const " +
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
      total[red[k]] = tv;
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
            std::to_string(bp.max_level) + " (grid barriers, cooperative launch)";
  return ks;
}

// ---- LITERAL --------------------------------------------------------------------

// chunk_box geometry (reference schedule.cpp:52-76) for a materialised member
struct Box {
  std::vector<std::string> lo;
  std::vector<int64_t> len;
};

Box chunk_box(Emitter& em, const Node& n, const Stmt& s, const std::string& blk) {
  Box b;
  const int rank = n.rank();
  b.lo.assign(rank, "0");
  b.len = n.dims;
  if (rank == 0) return b;
  const int64_t sd = s.split_dim;
  const int64_t slice_len = n.dims[sd] / s.sword;
  std::string slice = em.ivar(Emitter::imod(blk, s.sword));
  std::string fixed = em.ivar(Emitter::idiv(blk, s.sword));
  b.lo[sd] = em.ivar(Emitter::imul(slice, slice_len));
  b.len[sd] = slice_len;
  if (s.sched == SFX_SCHED_ROW) {
    for (int64_t i = sd - 1; i >= 0; --i) {
      b.lo[i] = em.ivar(Emitter::imod(fixed, n.dims[i]));
      fixed = em.ivar(Emitter::idiv(fixed, n.dims[i]));
      b.len[i] = 1;
    }
  } else {
    for (int64_t i = rank - 1; i > sd; --i) {
      b.lo[i] = em.ivar(Emitter::imod(fixed, n.dims[i]));
      fixed = em.ivar(Emitter::idiv(fixed, n.dims[i]));
      b.len[i] = 1;
    }
  }
  return b;
}

KernelSource lower_literal(const Ctx& c) {
  KernelSource ks;
  ks.strategy = "literal";
  ks.entry = "sfx_lit_" + c.name;
  fill_common(c, ks);
  const Graph& g = c.g;
  const Program& p = c.p;
  // materialised members and their statements
  std::map<int, const Stmt*> mat;
  int64_t max_chunk = 1;
  for (const Stmt& s : p.stmts)
    if (s.kind == SFX_STMT_MATERIALIZE) {
      mat[s.instr] = &s;
      max_chunk = std::max(max_chunk, g.nodes[s.instr].numel() / p.blocks);
    }
  int B = static_cast<int>(std::min<int64_t>(256, std::max<int64_t>(32, (max_chunk + 31) / 32 * 32)));
  Emitter em(g, p, 1, c.wide);
  std::string sig = signature(c, em, ks.entry, B);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  int64_t staging = 0;  // extra smem for two-phase writes into an aliased buffer
  // ready-set simulation (reference exec.cpp:300-392): arena reads only of
  // members materialised earlier in this block and not overwritten since.
  std::set<int> ready;
  std::set<int> read_now;
  std::string blk = "blk";
  std::map<int, Box> boxes;
  em.resolve = [&](int node, const std::vector<Ix>& comps) -> std::string {
    if (!ready.count(node)) return "";
    read_now.insert(node);
    const Node& n = g.nodes[node];
    const Stmt& s = *mat.at(node);
    Box& b = boxes[node];
    std::vector<Ix> local(comps.size());
    std::string L = "0";
    for (size_t d = 0; d < comps.size(); ++d) {
      std::string off = b.lo[d] == "0" ? comps[d].e : "(" + comps[d].e + "-" + b.lo[d] + ")";
      L = Emitter::iadd(Emitter::imul(L, b.len[d]), off);
      if (!Emitter::is_lit(L)) L = em.ivar(L);
    }
    std::string v = em.fresh("s");
    const char* T = ctype(n.dtype);
    em.code->line(std::string("const ") + T + " " + v + " = ((const " + T + "*)(sfx_arena + " + fmt_i(s.offset) +
                  "))[" + L + "];");
    return v;
  };
  body.line("extern __shared__ __align__(16) unsigned char sfx_arena[];");
  body.line("for (" + it + " blk = blockIdx.x; blk < " + fmt_i(p.blocks) + "; blk += gridDim.x) {");
  body.indent++;
  em.push();
  for (const Stmt& s : p.stmts) {
    if (s.kind == SFX_STMT_BARRIER) {
      body.line("__syncthreads();");
      continue;
    }
    if (s.kind != SFX_STMT_MATERIALIZE) continue;
    const Node& n = g.nodes[s.instr];
    Box b = chunk_box(em, n, s, blk);
    const int64_t chunk = n.numel() / p.blocks;
    const char* T = ctype(n.dtype);
    // detect whether this write aliases a ready buffer it reads (two-phase commit)
    bool shared_dest = s.dest == SFX_DEST_SHARED;
    std::string stage;
    Code saved;
    read_now.clear();
    Code tmp;
    tmp.indent = body.indent + 1;
    Code* outer = em.code;
    // emit the element loop body into tmp first to learn which buffers it reads
    em.code = &tmp;
    em.push();
    std::string k = em.fresh("k");
    std::vector<Ix> local = em.from_linear(em.uni(k), b.len);
    std::vector<Ix> comps(n.rank());
    for (int d = 0; d < n.rank(); ++d) comps[d] = em.uni(em.ivar(Emitter::iadd(b.lo[d], local[d].e)));
    std::string v = em.value(s.instr, comps);
    bool hazard = false;
    if (shared_dest)
      for (int r : read_now) {
        const Stmt& rs = *mat.at(r);
        int64_t len = g.nodes[r].numel() / p.blocks * 4;
        if (rs.offset < s.offset + s.bytes && s.offset < rs.offset + len) hazard = true;
      }
    if (shared_dest) {
      if (hazard) {
        staging = std::max<int64_t>(staging, chunk * 4);
        tmp.line(std::string("((") + T + "*)(sfx_arena + " + fmt_i(p.arena_bytes) + "))[" + k + "] = " + v + ";");
      } else {
        tmp.line(std::string("((") + T + "*)(sfx_arena + " + fmt_i(s.offset) + "))[" + k + "] = " + v + ";");
      }
    } else {
      std::string lin = "0";
      for (int d = 0; d < n.rank(); ++d) lin = Emitter::iadd(Emitter::imul(lin, n.dims[d]), comps[d].e);
      tmp.line("out" + std::to_string(s.root_index) + "[" + lin + "] = " + v + ";");
    }
    em.pop();
    em.code = outer;
    body.line("for (" + it + " " + k + " = threadIdx.x; " + k + " < " + fmt_i(chunk) + "; " + k + " += " +
              std::to_string(B) + ") {");
    body.text += tmp.text;
    body.line("}");
    if (shared_dest && hazard) {
      body.line("__syncthreads();");
      body.line("for (" + it + " " + k + " = threadIdx.x; " + k + " < " + fmt_i(chunk) + "; " + k + " += " +
                std::to_string(B) + ")");
      body.line(std::string("  ((") + T + "*)(sfx_arena + " + fmt_i(s.offset) + "))[" + k + "] = ((" + T +
                "*)(sfx_arena + " + fmt_i(p.arena_bytes) + "))[" + k + "];");
    }
    if (shared_dest) {
      for (auto itr = ready.begin(); itr != ready.end();) {
        const Stmt& rs = *mat.at(*itr);
        int64_t len = g.nodes[*itr].numel() / p.blocks * 4;
        bool overlap = rs.offset < s.offset + s.bytes && s.offset < rs.offset + len;
        if (overlap && *itr != s.instr)
          itr = ready.erase(itr);
        else
          ++itr;
      }
      ready.insert(s.instr);
      boxes[s.instr] = b;
    }
  }
  body.line("__syncthreads();");
  em.pop();
  body.indent--;
  body.line("}");
  ks.code = assemble(sig, body);
  ks.block = B;
  ks.grid_x = std::min<int64_t>(p.blocks, static_cast<int64_t>(kNumSMs) * 16);
  ks.smem = static_cast<int>(p.arena_bytes + staging);
  ks.vector_width = 1;
  ks.note = "reference geometry: blocks=" + std::to_string(p.blocks) + " arena=" + std::to_string(p.arena_bytes) + "B";
  return ks;
}

}  // namespace

std::string choose_strategy(const Graph& g, int pi, std::string* why) {
  const Program& p = g.programs.at(pi);
  if (dot_alone(g, p)) return "dot";
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
  if (why) *why = reasons;
  return "literal";
}

// ---- template parameter cache -------------------------------------------------
//
// Persisted, PerfLibrary-style text (reference tuning.cpp:41-125 stores measured
// schedule costs the same way): one line per group signature
//   signature|rows_per_cta|threads_per_row|items_per_thread|pipe_ctas_per_sm|tuned_us|default_us|source
// where signature = <entry>-<fnv64 of the kernel the default options generate>.
// tools/autotune.py measures candidate template parameters per group on the
// B200 and writes the winners; lowering with default options looks the group up
// and re-lowers with the recorded parameters.  SFX_TEMPLATE_PARAMS=<file>
// overrides the location, SFX_TEMPLATE_PARAMS=0 disables the cache.
namespace {
struct TunedParams {
  int rows_per_cta = 0, threads_per_row = 0, items_per_thread = 0, pipe_ctas_per_sm = 0;
  std::string note;
};
const std::map<std::string, TunedParams>& template_params() {
  static std::map<std::string, TunedParams> m;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = std::getenv("SFX_TEMPLATE_PARAMS");
    if (e && e[0] == '0' && e[1] == 0) return;
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

KernelSource lower_program(const Graph& g, int pi, const sfx_compile_opts& o) {
  KernelSource ks = lower_program_raw(g, pi, o);
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(fnv1a64(ks.code)));
  const std::string sig = ks.entry + "-" + hex;
  if (default_knobs(o)) {
    auto it = template_params().find(sig);
    if (it != template_params().end()) {
      sfx_compile_opts t = o;
      t.rows_per_cta = it->second.rows_per_cta;
      t.threads_per_row = it->second.threads_per_row;
      t.items_per_thread = it->second.items_per_thread;
      t.pipe_ctas_per_sm = it->second.pipe_ctas_per_sm;
      ks = lower_program_raw(g, pi, t);
      ks.note += " [template_params: " + it->second.note + "]";
    }
  }
  ks.note += " sig=" + sig;
  return ks;
}

KernelSource lower_program_raw(const Graph& g, int pi, const sfx_compile_opts& o) {
  if (pi < 0 || pi >= static_cast<int>(g.programs.size())) throw Error(SFX_ERR_INVALID, "program index out of range");
  const Program& p = g.programs[pi];
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
      const int Vr = rp.C % 4 == 0 ? 4 : 1;
      if (rp.C / row_tpr(rp.C, Vr) > 64)
        ks = lower_row_mp(c, rp, o);  // longer than 1024 threads x 64 elements
      else if (pipe_ok && o.row_pipeline == 2)
        ks = lower_row_pipe(c, rp, staged, o);
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
      if (!analyze_colbc(c, &bp, &why)) throw Error(SFX_ERR_UNSUPPORTED, "colbc template not applicable: " + why);
      ks = lower_colbc(c, bp, o);
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
