#include "emit.hpp"

#include <cinttypes>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace sfx {

std::string fmt_f32(double v) {
  float f = static_cast<float>(v);  // constant_value: static_cast<float>(raw) (exec.cpp:220-221)
  if (!std::isfinite(f)) {
    uint32_t bits;
    std::memcpy(&bits, &f, 4);
    char buf[48];
    std::snprintf(buf, sizeof buf, "sfx_bits_f((int)0x%08xu)", bits);
    return buf;
  }
  char buf[64];
  std::snprintf(buf, sizeof buf, "%af", static_cast<double>(f));
  return buf;
}

std::string fmt_f64(double v) {
  if (!std::isfinite(v)) {
    if (std::isnan(v)) return "__longlong_as_double(0x7ff8000000000000ll)";
    return v > 0 ? "__longlong_as_double(0x7ff0000000000000ll)" : "__longlong_as_double((long long)0xfff0000000000000ull)";
  }
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", v);
  return buf;
}

std::string fmt_i(int64_t v) {
  char buf[32];
  if (v > INT_MAX || v < INT_MIN)
    std::snprintf(buf, sizeof buf, "%" PRId64 "ll", v);
  else
    std::snprintf(buf, sizeof buf, "%" PRId64, v);
  return buf;
}

const char* ctype(int dtype) { return dtype == SFX_F32 ? "float" : "int"; }

Emitter::Emitter(const Graph& g_, const Program& p_, int vec, bool wide_index)
    : g(g_), p(p_), V(vec), idx_t(wide_index ? "long long" : "int") {
  scopes_.emplace_back();
}

std::string Emitter::fresh(const char* prefix) { return std::string(prefix) + std::to_string(next_++); }
void Emitter::push() { scopes_.emplace_back(); }
void Emitter::pop() { scopes_.pop_back(); }

std::string Emitter::find(const std::string& key) const {
  for (auto it = scopes_.rbegin(); it != scopes_.rend(); ++it) {
    auto f = it->find(key);
    if (f != it->end()) return f->second;
  }
  return "";
}

void Emitter::bind(const std::string& key, const std::string& var) { scopes_.back()[key] = var; }

bool Emitter::is_lit(const std::string& s, int64_t* v) {
  if (s.empty()) return false;
  size_t i = 0;
  if (s[0] == '-') i = 1;
  if (i >= s.size()) return false;
  size_t end = s.size();
  if (end >= 2 && s.compare(end - 2, 2, "ll") == 0) end -= 2;
  for (size_t k = i; k < end; ++k)
    if (s[k] < '0' || s[k] > '9') return false;
  if (v) *v = std::stoll(s.substr(0, end));
  return true;
}

std::string Emitter::imul(const std::string& a, int64_t k) {
  int64_t v;
  if (k == 0) return "0";
  if (k == 1) return a;
  if (is_lit(a, &v)) return fmt_i(v * k);
  return "(" + a + "*" + fmt_i(k) + ")";
}

std::string Emitter::iadd(const std::string& a, const std::string& b) {
  int64_t x, y;
  bool la = is_lit(a, &x), lb = is_lit(b, &y);
  if (la && lb) return fmt_i(x + y);
  if (la && x == 0) return b;
  if (lb && y == 0) return a;
  return "(" + a + "+" + b + ")";
}

std::string Emitter::idiv(const std::string& a, int64_t k) {
  int64_t v;
  if (k == 1) return a;
  if (is_lit(a, &v)) return fmt_i(v / k);
  return "(" + a + "/" + fmt_i(k) + ")";
}

std::string Emitter::imod(const std::string& a, int64_t k) {
  int64_t v;
  if (k == 1) return "0";
  if (is_lit(a, &v)) return fmt_i(v % k);
  return "(" + a + "%" + fmt_i(k) + ")";
}

static bool is_ident(const std::string& s) {
  if (s.empty()) return false;
  if (!(std::isalpha(static_cast<unsigned char>(s[0])) || s[0] == '_')) return false;
  for (char c : s)
    if (!(std::isalnum(static_cast<unsigned char>(c)) || c == '_')) return false;
  return true;
}

std::string Emitter::ivar(const std::string& expr) {
  if (is_lit(expr) || is_ident(expr)) return expr;
  std::string key = "ix:" + expr;
  std::string v = find(key);
  if (!v.empty()) return v;
  v = fresh("i");
  code->line("const " + idx_t + " " + v + " = " + expr + ";");
  bind(key, v);
  return v;
}

Ix Emitter::lane_plus(const std::string& base) {
  Ix x;
  x.kind = IX_PLUS;
  x.base = base;
  x.e = lane == 0 ? base : ivar(iadd(base, std::to_string(lane)));
  return x;
}

// Row-major delinearisation (reference exec.cpp:124-131) with lane tracking.
std::vector<Ix> Emitter::from_linear(const Ix& lin, const std::vector<int64_t>& dims) {
  const int n = static_cast<int>(dims.size());
  std::vector<Ix> out(n);
  if (n == 0) return out;
  std::vector<int64_t> stride(n, 1);
  for (int k = n - 2; k >= 0; --k) stride[k] = stride[k + 1] * dims[k + 1];
  auto comp = [&](const std::string& L, int k) -> std::string {
    if (dims[k] == 1) return "0";
    std::string q = idiv(L, stride[k]);
    if (k > 0) q = imod(q, dims[k]);
    return ivar(q);
  };
  if (lin.kind == IX_UNI) {
    std::string L = ivar(lin.e);
    for (int k = 0; k < n; ++k) out[k] = uni(comp(L, k));
    return out;
  }
  if (lin.kind == IX_PLUS && V > 1 && dims[n - 1] % V == 0) {
    std::string B = ivar(lin.base);
    for (int k = 0; k < n - 1; ++k) out[k] = uni(comp(B, k));
    std::string lb = dims[n - 1] == 1 ? std::string("0") : ivar(n == 1 ? B : imod(B, dims[n - 1]));
    out[n - 1] = lane_plus(lb);
    return out;
  }
  std::string L = ivar(lin.e);
  for (int k = 0; k < n; ++k) {
    out[k].e = comp(L, k);
    out[k].base = out[k].e;
    out[k].kind = IX_CPLX;
  }
  return out;
}

// Row-major linearisation (reference exec.cpp:118-122) with lane tracking.
Ix Emitter::linearize(const std::vector<Ix>& comps, const std::vector<int64_t>& dims) {
  const int n = static_cast<int>(dims.size());
  if (n == 0) return uni("0");
  int plus_at = -1, nplus = 0;
  bool cplx = false;
  for (int k = 0; k < n; ++k) {
    if (comps[k].kind == IX_PLUS) {
      plus_at = k;
      ++nplus;
    }
    if (comps[k].kind == IX_CPLX) cplx = true;
  }
  auto lin_of = [&](bool use_base) {
    std::string L = "0";
    for (int k = 0; k < n; ++k) {
      const std::string& c = (use_base && comps[k].kind == IX_PLUS) ? comps[k].base : comps[k].e;
      L = iadd(imul(L, dims[k]), c);
      if (k + 1 < n && !is_lit(L)) L = ivar(L);
    }
    return L;
  };
  if (!cplx && nplus == 0) return uni(ivar(lin_of(false)));
  if (!cplx && nplus == 1 && plus_at == n - 1 && dims[n - 1] % V == 0) {
    std::string B = ivar(lin_of(true));
    return lane_plus(B);
  }
  Ix x;
  x.e = ivar(lin_of(false));
  x.base = x.e;
  x.kind = IX_CPLX;
  return x;
}

// A value held in shared memory for the current row (an input staged by TMA,
// or a member cached by an earlier pass over the row): `sp` points at the
// row's slice, `rb` is the linear index of its first element.
std::string Emitter::staged_load(int node, const std::vector<Ix>& comps) {
  const Node& n = g.nodes[node];
  Ix L = linearize(comps, n.dims);
  const auto& st = staged.at(node);
  const std::string& sp = st.first;
  const std::string& rb = st.second;
  if (L.kind == IX_PLUS && V == 4) {
    std::string key = "sld4:" + sp + ":" + L.base;
    std::string q = find(key);
    if (q.empty()) {
      q = fresh("q");
      code->line("const sfx_f4 " + q + " = sfx_lds4(" + sp + " + (" + L.base + " - " + rb + "));");
      bind(key, q);
      ++loads_vec;
    }
    static const char* xyzw[] = {".x", ".y", ".z", ".w"};
    return q + xyzw[lane];
  }
  std::string key = "sld:" + sp + ":" + L.e;
  std::string v = find(key);
  if (v.empty()) {
    v = fresh("v");
    code->line("const float " + v + " = " + sp + "[" + L.e + " - " + rb + "];");
    bind(key, v);
    ++loads_scalar;
  }
  return v;
}

std::string Emitter::load(int node, const std::vector<Ix>& comps) {
  const Node& n = g.nodes[node];
  auto pit = input_ptr.find(node);
  if (pit == input_ptr.end()) throw Error(SFX_ERR_EXEC, "missing external value " + n.id);
  const std::string& ptr = pit->second;
  auto tt = tiled.find(node);
  if (tt != tiled.end()) {  // transposed tile in shared memory
    const Tile& t = tt->second;
    std::string B = t.mb ? imod(comps[t.jb].e, t.mb) : comps[t.jb].e;
    std::string A = t.ma ? imod(idiv(comps[t.ja].e, t.sa), t.ma) : comps[t.ja].e;
    std::string addr;
    if (t.swz) {
      const std::string ra = ivar("(int)(" + A + " - " + t.a0 + ")"), rb = ivar("(int)(" + B + " - " + t.b0 + ")");
      addr = t.arr + "[" + ra + " * 64 + ((((" + rb + ") >> 2) ^ ((" + ra + " >> 2) & 7)) << 2) + ((" + rb + ") & 3)]";
    } else {
      addr = t.arr + "[" + B + " - " + t.b0 + "][" + A + " - " + t.a0 + "]";
    }
    std::string key = "tld:" + addr;
    std::string v = find(key);
    if (v.empty()) {
      v = fresh("v");
      code->line(std::string("const ") + ctype(n.dtype) + " " + v + " = " + addr + ";");
      bind(key, v);
    }
    return v;
  }
  if (staged.count(node)) return staged_load(node, comps);  // row staged in shared memory by TMA
  Ix L = linearize(comps, n.dims);
  if (L.kind == IX_PLUS && V == 4) {
    std::string key = "ld4:" + ptr + ":" + L.base;
    std::string q = find(key);
    if (q.empty()) {
      q = fresh("q");
      const char* vt = n.dtype == SFX_F32 ? "sfx_f4" : "sfx_i4";
      const char* fn = streaming.count(node) ? "sfx_ld4s" : "sfx_ld4";
      code->line(std::string("const ") + vt + " " + q + " = " + fn + "(" + ptr + " + " + L.base + ");");
      bind(key, q);
      ++loads_vec;
    }
    static const char* xyzw[] = {".x", ".y", ".z", ".w"};
    return q + xyzw[lane];
  }
  std::string key = "ld:" + ptr + ":" + L.e;
  std::string v = find(key);
  if (!v.empty()) return v;
  v = fresh("v");
  code->line(std::string("const ") + ctype(n.dtype) + " " + v + " = sfx_ld(" + ptr + " + " + L.e + ");");
  bind(key, v);
  ++loads_scalar;
  return v;
}

std::string Emitter::seq_fold(int reducer, int dtype, const std::string& acc, const std::string& v) {
  (void)dtype;
  switch (reducer) {
    case SFX_REDUCE_SUM: return "sfx_add(" + acc + ", " + v + ")";
    case SFX_REDUCE_MAX: return "sfx_max(" + acc + ", " + v + ")";
    default: return "sfx_min(" + acc + ", " + v + ")";
  }
}

// A group member whose value depends on a (non-degenerate) reduction of the group.
bool Emitter::reduce_dependent(int node) {
  auto it = reduce_dep_.find(node);
  if (it != reduce_dep_.end()) return it->second;
  bool r = false;
  if (p.is_member(node)) {
    const Node& n = g.nodes[node];
    r = n.op == SFX_OP_REDUCE;
    for (int op : n.operands) r = r || reduce_dependent(op);
  }
  return reduce_dep_[node] = r;
}

std::string Emitter::ew_expr(const Node& n, const std::vector<std::string>& a) {
  switch (n.kind) {
    case SFX_EW_ADD: return "sfx_add(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_SUB: return "sfx_sub(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_MUL: return "sfx_mul(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_MAX: return "sfx_max(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_MIN: return "sfx_min(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_NEG: return "sfx_neg(" + a[0] + ")";
    case SFX_EW_COMPARE: return "sfx_cmp(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_SELECT: return "sfx_sel(" + a[0] + ", " + a[1] + ", " + a[2] + ")";
    case SFX_EW_SCALE: {
      // float(x * double(s)) (exec.cpp:23).  When s is exactly a float the
      // double product of two floats is exact, so one fp32 multiply rounds
      // identically.
      if (n.dtype == SFX_F32 && static_cast<double>(static_cast<float>(n.scalar)) == n.scalar &&
          std::isfinite(n.scalar))
        return "sfx_scale_f(" + a[0] + ", " + fmt_f32(n.scalar) + ")";
      if (n.dtype == SFX_F32 && std::isfinite(n.scalar) && std::fabs(n.scalar) < 1e30 &&
          std::fabs(n.scalar) > 1e-30) {
        // s = hi + lo (two floats); fma(x, hi, x*lo) is x*s with one final
        // rounding of a value within 2^-48 relative of the exact product: the
        // same float as float(x*double(s)) except at near-midpoints (<= 1 ulp),
        // at FP32 instead of FP64/F2F throughput.
        // hi is s truncated toward zero, so lo has the sign of hi and
        // fma(+-inf, hi, +-inf*lo) stays +-inf (no NaN from opposite infinities).
        float hi = static_cast<float>(n.scalar);
        if (std::fabs(static_cast<double>(hi)) > std::fabs(n.scalar))
          hi = std::nextafter(hi, 0.0f);
        float lo = static_cast<float>(n.scalar - static_cast<double>(hi));
        return "sfx_scale_2f(" + a[0] + ", " + fmt_f32(hi) + ", " + fmt_f32(lo) + ")";
      }
      return "sfx_scale_d(" + a[0] + ", " + fmt_f64(n.scalar) + ")";
    }
    case SFX_EW_EXP: return "sfx_exp(" + a[0] + ")";
    case SFX_EW_LOG: return "sfx_log(" + a[0] + ")";
    case SFX_EW_DIVIDE: return "sfx_div(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_POWER: return "sfx_pow(" + a[0] + ", " + a[1] + ")";
    case SFX_EW_TANH: return "sfx_tanh(" + a[0] + ")";
    case SFX_EW_SQRT: return "sfx_sqrt(" + a[0] + ")";
    case SFX_EW_RSQRT: return "sfx_rsqrt(" + a[0] + ")";
  }
  throw Error(SFX_ERR_INVALID, "bad elementwise kind in " + n.id);
}

// In-register fold in the reference's order (exec.cpp:182-204): row-major over
// the reduced sub-space, first element initialises the accumulator.
std::string Emitter::reduce_loop(int node, const std::vector<Ix>& comps) {
  const Node& n = g.nodes[node];
  const Node& in = g.nodes[n.operands[0]];
  std::set<int64_t> rd(n.reduce_dims.begin(), n.reduce_dims.end());
  std::vector<int64_t> red;
  for (int d = 0; d < in.rank(); ++d)
    if (rd.count(d)) red.push_back(in.dims[d]);
  int64_t nred = 1;
  for (int64_t d : red) nred *= d;
  if (nred == 1) {  // a fold of one element is that element (exec.cpp:196-201)
    std::vector<Ix> oc(in.rank());
    for (int d = 0, o = 0; d < in.rank(); ++d) oc[d] = rd.count(d) ? uni("0") : comps[o++];
    return value(n.operands[0], oc);
  }
  std::string acc = fresh("a");
  std::string q = fresh("r");
  const char* T = ctype(n.dtype);
  code->line(std::string(T) + " " + acc + ";");
  code->line("for (" + idx_t + " " + q + " = 0; " + q + " < " + fmt_i(nred) + "; ++" + q + ") {");
  code->indent++;
  push();
  int saved_lane = lane;
  std::vector<Ix> rc = from_linear(uni(q), red);
  std::vector<Ix> oc(in.rank());
  for (int d = 0, o = 0, r = 0; d < in.rank(); ++d) oc[d] = rd.count(d) ? rc[r++] : comps[o++];
  std::string v = value(n.operands[0], oc);
  lane = saved_lane;
  code->line(acc + " = (" + q + " == 0) ? " + v + " : " + seq_fold(n.reducer, n.dtype, acc, v) + ";");
  pop();
  code->indent--;
  code->line("}");
  return acc;
}

// matmul_element (exec.cpp:84-100): acc starts at 0, then acc = acc + a*b over
// the contraction index in ascending order (two roundings per step, no FMA).
std::string Emitter::dot_loop(int node, const std::vector<Ix>& comps) {
  const Node& n = g.nodes[node];
  const Node& a = g.nodes[n.operands[0]];
  const int r = n.rank();
  const int64_t K = a.dims[r - 1];
  std::string acc = fresh("a");
  std::string q = fresh("k");
  code->line(std::string(ctype(n.dtype)) + " " + acc + " = " + (n.dtype == SFX_F32 ? "0.0f" : "0") + ";");
  code->line("for (" + idx_t + " " + q + " = 0; " + q + " < " + fmt_i(K) + "; ++" + q + ") {");
  code->indent++;
  push();
  int saved_lane = lane;
  std::vector<Ix> li(comps.begin(), comps.end()), ri(comps.begin(), comps.end());
  li[r - 1] = uni(q);
  ri[r - 2] = uni(q);
  std::string x = value(n.operands[0], li);
  std::string y = value(n.operands[1], ri);
  lane = saved_lane;
  code->line(acc + " = sfx_add(" + acc + ", sfx_mul(" + x + ", " + y + "));");
  pop();
  code->indent--;
  code->line("}");
  return acc;
}

std::string Emitter::value(int node, const std::vector<Ix>& comps) {
  const Node& n = g.nodes[node];
  if (n.is_splat()) return n.dtype == SFX_F32 ? fmt_f32(n.literal[0]) : fmt_i(static_cast<int32_t>(n.literal[0]));
  std::string key = "v" + std::to_string(node);
  for (const Ix& c : comps) key += "|" + c.e;
  std::string hit = find(key);
  if (!hit.empty()) return hit;

  std::string result;
  if (p.is_member(node) && staged.count(node)) {  // cached in shared memory by an earlier pass
    result = staged_load(node, comps);
    bind(key, result);
    return result;
  }
  if (!p.is_member(node)) {
    result = load(node, comps);
    bind(key, result);
    return result;
  }
  if (resolve) {
    result = resolve(node, comps);
    if (!result.empty()) {
      bind(key, result);
      return result;
    }
  }
  const char* T = ctype(n.dtype);
  switch (n.op) {
    case SFX_OP_ELEMENTWISE: {
      std::vector<std::string> a;
      for (int op : n.operands) a.push_back(value(op, comps));
      result = fresh("v");
      if (rcp_reduced_divisors && n.kind == SFX_EW_DIVIDE && n.dtype == SFX_F32 && reduce_dependent(n.operands[1])) {
        const std::string key = "rcp:" + a[1];
        std::string r = find(key);
        if (r.empty()) {
          r = fresh("rcp");
          code->line("const float " + r + " = sfx_rcp(" + a[1] + ");");
          bind(key, r);
        }
        code->line(std::string("const ") + T + " " + result + " = sfx_div_rc(" + a[0] + ", " + a[1] + ", " + r + ");");
        break;
      }
      code->line(std::string("const ") + T + " " + result + " = " + ew_expr(n, a) + ";");
      break;
    }
    case SFX_OP_RESHAPE:
    case SFX_OP_BITCAST: {
      const Node& in = g.nodes[n.operands[0]];
      Ix L = linearize(comps, n.dims);
      std::string v = value(n.operands[0], from_linear(L, in.dims));
      if (in.dtype == n.dtype) {
        result = v;
      } else {
        result = fresh("v");
        code->line(std::string("const ") + T + " " + result + " = " +
                   (n.dtype == SFX_F32 ? "sfx_bits_f(" : "sfx_bits_i(") + v + ");");
      }
      break;
    }
    case SFX_OP_TRANSPOSE: {
      std::vector<Ix> oc(comps.size());
      for (size_t i = 0; i < comps.size(); ++i) oc[n.perm[i]] = comps[i];
      result = value(n.operands[0], oc);
      break;
    }
    case SFX_OP_BROADCAST: {
      std::vector<Ix> oc(n.dim_map.size());
      for (size_t j = 0; j < n.dim_map.size(); ++j) oc[j] = comps[n.dim_map[j]];
      result = value(n.operands[0], oc);
      break;
    }
    case SFX_OP_REDUCE:
      result = reduce_loop(node, comps);
      break;
    case SFX_OP_BATCH_MATMUL:
      result = dot_loop(node, comps);
      break;
    default:
      throw Error(SFX_ERR_INVALID, "cannot evaluate " + n.id + " inside a group");
  }
  bind(key, result);
  return result;
}

}  // namespace sfx
