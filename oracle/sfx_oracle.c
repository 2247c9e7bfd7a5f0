/* TEST INFRASTRUCTURE — see sfx_oracle.h.  Restates reference
 * proj/src/exec.cpp (interpret / compute_element) in C over include/sfx.h
 * descriptors.  Build: oracle/Makefile (-O2 -ffp-contract=off, glibc libm, the
 * same libm the reference links). */
#include "sfx_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* sfx_oracle_error(void) { return g_err; }

static int fail(const char* what, const char* id) {
  snprintf(g_err, sizeof g_err, "%s%s%s", what, id ? " " : "", id ? id : "");
  return 1;
}

static int64_t numel(const sfx_instr* s) {
  int64_t n = 1;
  for (int i = 0; i < s->rank; ++i) n *= s->dims[i];
  return n;
}

/* exec.cpp:124-131 */
static void delin(int64_t lin, const int64_t* dims, int rank, int64_t* idx) {
  for (int d = rank - 1; d >= 0; --d) {
    idx[d] = lin % dims[d];
    lin /= dims[d];
  }
}

/* exec.cpp:118-122 */
static int64_t linz(const int64_t* idx, const int64_t* dims, int rank) {
  int64_t l = 0;
  for (int d = 0; d < rank; ++d) l = l * dims[d] + idx[d];
  return l;
}

typedef struct {
  const sfx_graph_desc* g;
  void* const* out;  /* caller buffers */
  double** dv;       /* mode 1: f32 nodes in double */
  int mode;
} Ctx;

/* ---- reference scalar semantics, fp32 (exec.cpp:18-65) ---- */
static float f_max(float x, float y) { return x < y ? y : x; } /* std::max */
static float f_min(float x, float y) { return y < x ? y : x; } /* std::min */

static float ew_f32(int kind, float x, float y, float z, double scalar) {
  switch (kind) {
    case SFX_EW_ADD: return x + y;
    case SFX_EW_SUB: return x - y;
    case SFX_EW_MUL: return x * y;
    case SFX_EW_MAX: return f_max(x, y);
    case SFX_EW_MIN: return f_min(x, y);
    case SFX_EW_NEG: return -x;
    case SFX_EW_COMPARE: return x > y ? 1.0f : 0.0f;
    case SFX_EW_SELECT: return x != 0.0f ? y : z; /* exec.cpp:145-148 */
    case SFX_EW_SCALE: return (float)(x * scalar); /* exec.cpp:23 */
    case SFX_EW_EXP: return expf(x);
    case SFX_EW_LOG: return logf(x);
    case SFX_EW_DIVIDE: return x / y;
    case SFX_EW_POWER: return powf(x, y);
    case SFX_EW_TANH: return tanhf(x);
    case SFX_EW_SQRT: return sqrtf(x);
    case SFX_EW_RSQRT: return 1.0f / sqrtf(x); /* exec.cpp:28 */
  }
  return 0.0f;
}

static double d_max(double x, double y) { return x < y ? y : x; }
static double d_min(double x, double y) { return y < x ? y : x; }

static double ew_f64(int kind, double x, double y, double z, double scalar) {
  switch (kind) {
    case SFX_EW_ADD: return x + y;
    case SFX_EW_SUB: return x - y;
    case SFX_EW_MUL: return x * y;
    case SFX_EW_MAX: return d_max(x, y);
    case SFX_EW_MIN: return d_min(x, y);
    case SFX_EW_NEG: return -x;
    case SFX_EW_COMPARE: return x > y ? 1.0 : 0.0;
    case SFX_EW_SELECT: return x != 0.0 ? y : z;
    case SFX_EW_SCALE: return x * scalar;
    case SFX_EW_EXP: return exp(x);
    case SFX_EW_LOG: return log(x);
    case SFX_EW_DIVIDE: return x / y;
    case SFX_EW_POWER: return pow(x, y);
    case SFX_EW_TANH: return tanh(x);
    case SFX_EW_SQRT: return sqrt(x);
    case SFX_EW_RSQRT: return 1.0 / sqrt(x);
  }
  return 0.0;
}

/* i32 (exec.cpp:32-37, 55-63): two's-complement wrap as on the reference's
 * x86-64 build; scale = static_cast<int32_t>(x * scalar) -> cvttsd2si, which
 * yields INT_MIN for NaN / out-of-range. */
static int32_t i_scale(int32_t x, double s) {
  double p = (double)x * s;
  if (!(p > -2147483649.0 && p < 2147483648.0)) return (int32_t)0x80000000u;
  return (int32_t)p;
}

static int32_t ew_i32(int kind, int32_t x, int32_t y, int32_t z, double scalar) {
  switch (kind) {
    case SFX_EW_ADD: return (int32_t)((uint32_t)x + (uint32_t)y);
    case SFX_EW_SUB: return (int32_t)((uint32_t)x - (uint32_t)y);
    case SFX_EW_MUL: return (int32_t)((uint32_t)x * (uint32_t)y);
    case SFX_EW_MAX: return x < y ? y : x;
    case SFX_EW_MIN: return y < x ? y : x;
    case SFX_EW_NEG: return (int32_t)(0u - (uint32_t)x);
    case SFX_EW_COMPARE: return x > y ? 1 : 0;
    case SFX_EW_SELECT: return x != 0 ? y : z;
    case SFX_EW_SCALE: return i_scale(x, scalar);
  }
  return 0;
}

static int is_f32(const sfx_instr* s) { return s->dtype == SFX_F32; }

/* accessors: element e of node k, as float/double/int */
static float getf(Ctx* c, int k, int64_t e) { return ((const float*)c->out[k])[e]; }
static double getd(Ctx* c, int k, int64_t e) {
  return c->mode == 1 ? c->dv[k][e] : (double)((const float*)c->out[k])[e];
}
static int32_t geti(Ctx* c, int k, int64_t e) { return ((const int32_t*)c->out[k])[e]; }

static void setf(Ctx* c, int k, int64_t e, float v) { ((float*)c->out[k])[e] = v; }
static void setd(Ctx* c, int k, int64_t e, double v) { c->dv[k][e] = v; }
static void seti(Ctx* c, int k, int64_t e, int32_t v) { ((int32_t*)c->out[k])[e] = v; }

/* copy element `src_e` of node `src` into element `dst_e` of node `dst` (same dtype) */
static void mov(Ctx* c, int dst, int64_t dst_e, int src, int64_t src_e) {
  const sfx_instr* s = &c->g->instrs[dst];
  if (!is_f32(s)) seti(c, dst, dst_e, geti(c, src, src_e));
  else if (c->mode == 1) setd(c, dst, dst_e, getd(c, src, src_e));
  else setf(c, dst, dst_e, getf(c, src, src_e));
}

static int eval(Ctx* c, int k) {
  const sfx_graph_desc* g = c->g;
  const sfx_instr* s = &g->instrs[k];
  const int64_t n = numel(s);
  int64_t idx[SFX_MAX_RANK], in_idx[SFX_MAX_RANK];
  switch (s->opcode) {
    case SFX_OP_PARAMETER:
      if (!c->out[k]) return fail("missing input for parameter", s->id);
      if (c->mode == 1 && is_f32(s))
        for (int64_t e = 0; e < n; ++e) c->dv[k][e] = getf(c, k, e);
      return 0;
    case SFX_OP_CONSTANT: /* constant_value, exec.cpp:213-229 */
      if (s->n_literal != 1 && s->n_literal != n) return fail("constant literal size mismatch for", s->id);
      for (int64_t e = 0; e < n; ++e) {
        double raw = s->literal[s->n_literal == 1 ? 0 : e];
        if (!is_f32(s)) seti(c, k, e, (int32_t)raw);
        else if (c->mode == 1) setd(c, k, e, (double)(float)raw);
        else setf(c, k, e, (float)raw);
      }
      return 0;
    case SFX_OP_ELEMENTWISE: {
      int a = s->operands[0], b = s->n_operands > 1 ? s->operands[1] : a, z = s->n_operands > 2 ? s->operands[2] : a;
      if (!is_f32(s)) {
        for (int64_t e = 0; e < n; ++e)
          seti(c, k, e, ew_i32(s->kind, geti(c, a, e), geti(c, b, e), geti(c, z, e), s->scalar));
      } else if (c->mode == 1) {
        for (int64_t e = 0; e < n; ++e)
          setd(c, k, e, ew_f64(s->kind, getd(c, a, e), getd(c, b, e), getd(c, z, e), s->scalar));
      } else {
        for (int64_t e = 0; e < n; ++e)
          setf(c, k, e, ew_f32(s->kind, getf(c, a, e), getf(c, b, e), getf(c, z, e), s->scalar));
      }
      return 0;
    }
    case SFX_OP_RESHAPE: /* exec.cpp:153-156: same linear order */
      for (int64_t e = 0; e < n; ++e) mov(c, k, e, s->operands[0], e);
      return 0;
    case SFX_OP_BITCAST: { /* exec.cpp:157-171 */
      const sfx_instr* in = &g->instrs[s->operands[0]];
      if (in->dtype == s->dtype) {
        for (int64_t e = 0; e < n; ++e) mov(c, k, e, s->operands[0], e);
      } else if (is_f32(s)) {
        for (int64_t e = 0; e < n; ++e) {
          int32_t bits = geti(c, s->operands[0], e);
          float f;
          memcpy(&f, &bits, 4);
          if (c->mode == 1) setd(c, k, e, f); else setf(c, k, e, f);
        }
      } else {
        for (int64_t e = 0; e < n; ++e) {
          float f = c->mode == 1 ? (float)getd(c, s->operands[0], e) : getf(c, s->operands[0], e);
          int32_t bits;
          memcpy(&bits, &f, 4);
          seti(c, k, e, bits);
        }
      }
      return 0;
    }
    case SFX_OP_TRANSPOSE: { /* exec.cpp:172-176 */
      const sfx_instr* in = &g->instrs[s->operands[0]];
      for (int64_t e = 0; e < n; ++e) {
        delin(e, s->dims, s->rank, idx);
        for (int i = 0; i < s->rank; ++i) in_idx[s->permutation[i]] = idx[i];
        mov(c, k, e, s->operands[0], linz(in_idx, in->dims, in->rank));
      }
      return 0;
    }
    case SFX_OP_BROADCAST: { /* exec.cpp:177-181 */
      const sfx_instr* in = &g->instrs[s->operands[0]];
      for (int64_t e = 0; e < n; ++e) {
        delin(e, s->dims, s->rank, idx);
        for (int j = 0; j < s->n_dim_map; ++j) in_idx[j] = idx[s->broadcast_dim_map[j]];
        mov(c, k, e, s->operands[0], linz(in_idx, in->dims, in->rank));
      }
      return 0;
    }
    case SFX_OP_REDUCE: { /* exec.cpp:182-204 + reduce_fold :67-74 */
      const int src = s->operands[0];
      const sfx_instr* in = &g->instrs[src];
      int red[SFX_MAX_RANK] = {0};
      for (int j = 0; j < s->n_reduce_dims; ++j) red[s->reduce_dims[j]] = 1;
      int64_t stride[SFX_MAX_RANK];
      stride[in->rank - 1] = 1;
      for (int d = in->rank - 2; d >= 0; --d) stride[d] = stride[d + 1] * in->dims[d + 1];
      int rdim[SFX_MAX_RANK], nr = 0;
      for (int d = 0; d < in->rank; ++d)
        if (red[d]) rdim[nr++] = d;
      for (int64_t e = 0; e < n; ++e) {
        delin(e, s->dims, s->rank, idx);
        int64_t base = 0;
        for (int d = 0, o = 0; d < in->rank; ++d)
          if (!red[d]) base += idx[o++] * stride[d];
        int64_t ri[SFX_MAX_RANK] = {0};
        int64_t off = base;
        float af = 0.0f;
        double ad = 0.0;
        int32_t ai = 0;
        int first = 1;
        for (;;) {
          if (!is_f32(s)) {
            int32_t v = geti(c, src, off);
            if (first) ai = v;
            else if (s->reducer == SFX_REDUCE_SUM) ai = (int32_t)((uint32_t)ai + (uint32_t)v);
            else if (s->reducer == SFX_REDUCE_MAX) ai = ai < v ? v : ai;
            else ai = v < ai ? v : ai;
          } else if (c->mode == 1) {
            double v = getd(c, src, off);
            if (first) ad = v;
            else if (s->reducer == SFX_REDUCE_SUM) ad = ad + v;
            else if (s->reducer == SFX_REDUCE_MAX) ad = d_max(ad, v);
            else ad = d_min(ad, v);
          } else {
            float v = getf(c, src, off);
            if (first) af = v;
            else if (s->reducer == SFX_REDUCE_SUM) af = af + v;
            else if (s->reducer == SFX_REDUCE_MAX) af = f_max(af, v);
            else af = f_min(af, v);
          }
          first = 0;
          /* advance(red_index, red_dims), exec.cpp:76-82 */
          int q = nr - 1;
          for (; q >= 0; --q) {
            int d = rdim[q];
            off += stride[d];
            if (++ri[q] < in->dims[d]) break;
            off -= stride[d] * in->dims[d];
            ri[q] = 0;
          }
          if (q < 0) break;
        }
        if (!is_f32(s)) seti(c, k, e, ai);
        else if (c->mode == 1) setd(c, k, e, ad);
        else setf(c, k, e, af);
      }
      return 0;
    }
    case SFX_OP_BATCH_MATMUL:
    case SFX_OP_LIBRARY_CALL: { /* matmul_element, exec.cpp:84-100 */
      const sfx_instr* lhs = &g->instrs[s->operands[0]];
      const sfx_instr* rhs = &g->instrs[s->operands[1]];
      if (s->opcode == SFX_OP_LIBRARY_CALL && (s->kind != SFX_CALLEE_MATMUL || s->n_operands != 2))
        return fail("library call is not executable:", s->id); /* exec.cpp:207-209 */
      int r = s->rank;
      int64_t K = lhs->dims[lhs->rank - 1];
      for (int64_t e = 0; e < n; ++e) {
        delin(e, s->dims, r, idx);
        int64_t li[SFX_MAX_RANK], ri[SFX_MAX_RANK];
        memcpy(li, idx, sizeof(int64_t) * r);
        memcpy(ri, idx, sizeof(int64_t) * r);
        float af = 0.0f;
        double ad = 0.0;
        int32_t ai = 0;
        for (int64_t q = 0; q < K; ++q) {
          li[r - 1] = q;
          ri[r - 2] = q;
          int64_t lo = linz(li, lhs->dims, r), ro = linz(ri, rhs->dims, r);
          if (!is_f32(s)) ai = (int32_t)((uint32_t)ai + (uint32_t)geti(c, s->operands[0], lo) * (uint32_t)geti(c, s->operands[1], ro));
          else if (c->mode == 1) ad += getd(c, s->operands[0], lo) * getd(c, s->operands[1], ro);
          else {
            float p = getf(c, s->operands[0], lo) * getf(c, s->operands[1], ro);
            af = af + p;
          }
        }
        if (!is_f32(s)) seti(c, k, e, ai);
        else if (c->mode == 1) setd(c, k, e, ad);
        else setf(c, k, e, af);
      }
      return 0;
    }
  }
  return fail("unknown opcode for", s->id);
}

int sfx_oracle_interpret(const sfx_graph_desc* g, void* const* values, int mode) {
  g_err[0] = 0;
  const int N = g->n_instrs;
  Ctx c = {g, values, NULL, mode};
  int* pending = calloc(N, sizeof(int));
  int* order = malloc(sizeof(int) * (N + 1));
  int rc = 0;
  if (mode == 1) {
    c.dv = calloc(N, sizeof(double*));
    for (int k = 0; k < N; ++k)
      if (is_f32(&g->instrs[k])) c.dv[k] = malloc(sizeof(double) * (numel(&g->instrs[k]) + 1));
  }
  /* topological order (any valid order gives the same values) */
  for (int k = 0; k < N; ++k) {
    for (int a = 0; a < g->instrs[k].n_operands; ++a) {
      int dup = 0;
      for (int b = 0; b < a; ++b) dup |= g->instrs[k].operands[b] == g->instrs[k].operands[a];
      if (!dup) pending[k]++;
    }
  }
  int head = 0, tail = 0;
  for (int k = 0; k < N; ++k)
    if (!pending[k]) order[tail++] = k;
  while (head < tail) {
    int v = order[head++];
    for (int k = 0; k < N; ++k) {
      const sfx_instr* s = &g->instrs[k];
      int uses = 0;
      for (int a = 0; a < s->n_operands; ++a) uses |= s->operands[a] == v;
      if (uses && --pending[k] == 0) order[tail++] = k;
    }
  }
  if (tail != N) {
    rc = fail("graph contains a cycle", NULL);
    goto done;
  }
  for (int i = 0; i < N && !rc; ++i) rc = eval(&c, order[i]);
  if (!rc && mode == 1)
    for (int k = 0; k < N; ++k)
      if (c.dv[k] && g->instrs[k].opcode != SFX_OP_PARAMETER) {
        int64_t n = numel(&g->instrs[k]);
        for (int64_t e = 0; e < n; ++e) ((float*)values[k])[e] = (float)c.dv[k][e];
      }
done:
  if (c.dv) {
    for (int k = 0; k < N; ++k) free(c.dv[k]);
    free(c.dv);
  }
  free(pending);
  free(order);
  return rc;
}

/* FNV-1a over a byte range (the hash ref_tool prints for reference outputs). */
uint64_t sfx_oracle_fnv1a(const void* data, uint64_t n, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (uint64_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

/* Input stream of sfx_gen.h, elements [offset, offset+n) (fast path for the
 * full-size parity tests; numpy restates the same stream in tests/sfx_testlib.py). */
#include "sfx_gen.h"
void sfx_oracle_gen(uint64_t seed, uint64_t tensor_index, int is_i32, float lo, float hi, void* out, int64_t n,
                    int64_t offset) {
  uint64_t key = sfx_gen_key(seed, tensor_index);
  float span = hi - lo;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = sfx_splitmix64(key + (uint64_t)(offset + i));
    if (is_i32) {
      ((int32_t*)out)[i] = 1 + (int32_t)(h >> 62);
    } else {
      float u = (float)(h >> 40) * (1.0f / 16777216.0f);
      float p = span * u;
      ((float*)out)[i] = lo + p;
    }
  }
}
