// Unfused instructions and matmuls.  The reference planner leaves some
// instructions out of every group (fusion.cpp:259-263): the fusion barriers
// (BatchMatMul when fuse_dot is off, LibraryCall; span.cpp:35-36) and stray
// shape ops; run_compiled evaluates them with eval_dense
// (pipeline.cpp:124-127).  barrier_program() wraps each in a one-member
// program so it runs as one kernel like any group (map/row/col/literal
// templates); matmuls get the kernel below, which follows matmul_element
// (exec.cpp:84-100):
//
//   out[b, m, n] = ((0 + A[b,m,0]*B[b,0,n]) + A[b,m,1]*B[b,1,n]) + ...
//
// in fp32 with one rounding per multiply and per add (no FMA), i32 wrapping.
// One kernel per barrier: a register-tiled SIMT GEMM (BM x BN output tile per
// CTA, TM x TN per thread, BK-deep shared-memory stages, double-buffered).
// Every output keeps its own accumulator and visits k in ascending order, so
// the result is bit-identical to the reference's sequential loop whatever the
// tiling; the zero padding of a ragged last k-stage adds +0 products, which is
// exact because an accumulator that starts at +0 can never be -0.
//
// Tensor cores are deliberately not used here: tcgen05 kinds (tf32/bf16/f16)
// round the operands, and a split-precision emulation would change the sum
// order; the reference's value is defined by the sequential fp32 loop.
#include <algorithm>
#include <cstdlib>
#include <cctype>
#include <map>
#include <set>
#include <sstream>

#include "emit.hpp"
#include "lower.hpp"

namespace sfx {

Program barrier_program(const Graph& g, int node) {
  const Node& n = g.nodes[node];
  Program p;
  p.members = {node};
  p.member_set = {node};
  p.roots = {node};
  p.fusion_root = node;
  p.barrier = true;
  std::set<int> ext(n.operands.begin(), n.operands.end());
  p.externals.assign(ext.begin(), ext.end());
  std::sort(p.externals.begin(), p.externals.end(), [&](int a, int b) { return g.nodes[a].id < g.nodes[b].id; });
  for (int e : p.externals)
    if (!g.nodes[e].is_splat()) p.inputs.push_back(e);
  // A plan for the literal tier: one block per index of the leading dim
  // (a row schedule, schedule.cpp:52-76), the member written straight to the
  // output.  The map/row/col templates do not read it.
  Stmt st;
  st.kind = SFX_STMT_MATERIALIZE;
  st.instr = node;
  st.sched = SFX_SCHED_ROW;
  st.split_dim = 0;
  st.sword = n.rank() > 0 ? n.dims[0] : 1;
  st.dest = SFX_DEST_OUTPUT;
  st.root_index = 0;
  p.stmts.push_back(st);
  p.blocks = st.sword;
  p.block_threads = 256;
  return p;
}

// SFX_DOT_PACKED=0: the FMUL + FADD kernel for every matmul (A/B)
bool dot_packed() {
  const char* e = std::getenv("SFX_DOT_PACKED");
  return !(e && e[0] == '0');
}

bool is_matmul(const Node& n) { return n.op == SFX_OP_BATCH_MATMUL || n.op == SFX_OP_LIBRARY_CALL; }

bool dot_alone(const Graph& g, const Program& p) {
  return p.members.size() == 1 && p.roots.size() == 1 && p.roots[0] == p.members[0] &&
         is_matmul(g.nodes[p.members[0]]);
}

namespace {

std::string subst(std::string s, const std::vector<std::pair<std::string, std::string>>& kv) {
  for (const auto& [k, v] : kv) {
    size_t pos = 0;
    while ((pos = s.find(k, pos)) != std::string::npos) {
      s.replace(pos, k.size(), v);
      pos += v.size();
    }
  }
  return s;
}

const char* kDotKernel = R"SFXDOT(
#define BM $BM
#define BN $BN
#define BK 16
#define TM $TM
#define TN $TN
#define NT ((BM / TM) * (BN / TN))
#define LA ((BM * BK) / NT)
#define LB ((BK * BN) / NT)
typedef $T T;
typedef $T4 T4;

extern "C" __global__ void __launch_bounds__(NT) $ENTRY($PARAMS) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const long long M = $M, N = $N, K = $K;
  __shared__ __align__(16) T As[2][BK][BM + 4];
  __shared__ __align__(16) T Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  long long t = blockIdx.x;
  const long long nb = t % $TILES_N;
  t /= $TILES_N;
  const long long mb = t % $TILES_M;
  const long long b = t / $TILES_M;
  const long long m0 = mb * BM, n0 = nb * BN;
  T ra[LA], rb[LB];
  auto fetch = [&](long long k0) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = tid + i * NT, row = e / BK, kk = e % BK;
      const long long m = m0 + row, k = k0 + kk;
      ra[i] = (m < M && k < K) ? $LOAD_A(b * M * K + m * K + k) : T(0);
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = tid + i * NT, kk = e / BN, col = e % BN;
      const long long k = k0 + kk, n = n0 + col;
      rb[i] = (k < K && n < N) ? $LOAD_B(b * K * N + k * N + n) : T(0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = tid + i * NT;
      As[buf][e % BK][e / BK] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = tid + i * NT;
      Bs[buf][e / BN][e % BN] = rb[i];
    }
  };
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (long long k0 = 0; k0 < K; k0 += BK) {
    const bool more = k0 + BK < K;
    if (more) fetch(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], v[TN];
#if TM % 4 == 0
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        const T4 q = *reinterpret_cast<const T4*>(&As[buf][kk][ty * TM + i]);
        a[i] = q.x; a[i + 1] = q.y; a[i + 2] = q.z; a[i + 3] = q.w;
      }
#else
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
#endif
#if TN % 4 == 0
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        const T4 q = *reinterpret_cast<const T4*>(&Bs[buf][kk][tx * TN + j]);
        v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
      }
#else
#pragma unroll
      for (int j = 0; j < TN; ++j) v[j] = Bs[buf][kk][tx * TN + j];
#endif
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = sfx_add(acc[i][j], sfx_mul(a[i], v[j]));
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const long long m = m0 + ty * TM + i;
    if (m >= M) continue;
    T* row = out0 + b * M * N + m * N;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const long long n = n0 + tx * TN + j;
      if (n < N) row[n] = acc[i][j];
    }
  }
}
)SFXDOT";

// The large-tile f32 variant (M, N >= 128, K and N multiples of 4, both
// operands in memory): 128x128 output tile per CTA, 8x8 per thread, 32-deep k
// stages, a 3-stage cp.async pipeline (A kept [m][k] as in memory, B [k][n]:
// no register staging, no transposing stores), and the products and sums in
// PACKED pairs on Blackwell's fp32x2 datapath:
//   t = fma.rn.f32x2(a, b, Z)     one rounding: fl(a*b + 0) = fl(a*b)
//   acc = add.rn.f32x2(acc, t)    one rounding: the reference's acc + a*b
// Z is a zero ptxas cannot see (read from %dynamic_smem_size >> 20 at run
// time), so it can neither turn the fma into a mul nor contract mul + add into
// one FFMA2 (which it does for mul.rn.f32x2 + add.rn.f32x2).  A -0 product
// becomes +0, which is harmless: an accumulator that starts at +0 never becomes
// -0, and adding +-0 to any other value returns it unchanged.  Measured
// bit-identical to FMUL+FADD on signed zeros, subnormals, infinities and NaN
// (tools/micro/fmul2.cu), and ~9% more multiply-adds per issue slot.
const char* kDotKernel2 = R"SFXDOT(
#define BM 128
#define BN $BN
#define TN $TN
#define BK 32
#define NS 3
#define NT 256
#define APAD (BK + 4)
#define BPAD (BN + 4)
typedef unsigned long long u64;
__device__ __forceinline__ u64 sfx_pk2(float x, float y) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void sfx_cp16z(void* smem, const void* gmem, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(sfx_smem_u32(smem)), "l"(gmem), "r"(ok ? 16 : 0)
               : "memory");
}

extern "C" __global__ void __launch_bounds__(NT, 2) $ENTRY($PARAMS) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const long long M = $M, N = $N, K = $K;
  extern __shared__ __align__(16) float sfx_dsm[];
  float* As = sfx_dsm;                     // [NS][BM][APAD]
  float* Bs = sfx_dsm + NS * BM * APAD;    // [NS][BK][BPAD]
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  long long t = blockIdx.x;
  const long long nb = t % $TILES_N;
  t /= $TILES_N;
  const long long mb = t % $TILES_M;
  const long long b = t / $TILES_M;
  const long long m0 = mb * BM, n0 = nb * BN;
  const float* Ab = $A + b * M * K;
  const float* Bb = $B + b * K * N;
  unsigned dsz;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
  const float zf = __uint_as_float(dsz >> 20);  // +0.0f at run time
  const u64 Z = sfx_pk2(zf, zf);
  // one stage: A [BM x BK] = 1024 16-byte chunks, B [BK x BN] = 1024; 4 + 4 per thread
  auto load = [&](long long k0, int st) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * NT, row = e / (BK / 4), kq = e % (BK / 4);
      const long long m = m0 + row, k = k0 + kq * 4;
      const bool ok = m < M && k < K;
      sfx_cp16z(As + (st * BM + row) * APAD + kq * 4, ok ? Ab + m * K + k : Ab, ok);
    }
#pragma unroll
    for (int i = 0; i < BK * BN / 4 / NT; ++i) {
      const int e = tid + i * NT, kk = e / (BN / 4), nq = e % (BN / 4);
      const long long k = k0 + kk, n = n0 + nq * 4;
      const bool ok = k < K && n < N;
      sfx_cp16z(Bs + (st * BK + kk) * BPAD + nq * 4, ok ? Bb + k * N + n : Bb, ok);
    }
  };
  u64 acc[8][TN / 2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TN / 2; ++j) acc[i][j] = 0ull;  // +0.0f pairs
  const long long nk = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nk) load((long long)s * BK, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (long long ks = 0; ks < nk; ++ks) {
    asm volatile("cp.async.wait_group %0;" :: "n"(NS - 2) : "memory");
    __syncthreads();  // stage ks landed for every thread; stage ks-1 is free
    if (ks + NS - 1 < nk) load((ks + NS - 1) * BK, (int)((ks + NS - 1) % NS));
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int st = (int)(ks % NS);
    const float* as = As + (st * BM + ty * 8) * APAD;
    const float* bs = Bs + st * BK * BPAD + tx * TN;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      float4 a4[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a4[i] = *reinterpret_cast<const float4*>(as + i * APAD + k4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        u64 bp[TN / 2];
#pragma unroll
        for (int h = 0; h < TN / 4; ++h) {
          const float4 b4 = *reinterpret_cast<const float4*>(bs + (k4 + q) * BPAD + 4 * h);
          bp[2 * h] = sfx_pk2(b4.x, b4.y);
          bp[2 * h + 1] = sfx_pk2(b4.z, b4.w);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float av = q == 0 ? a4[i].x : q == 1 ? a4[i].y : q == 2 ? a4[i].z : a4[i].w;
          const u64 ap = sfx_pk2(av, av);
#pragma unroll
          for (int j = 0; j < TN / 2; ++j) {
            u64 pr;
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pr) : "l"(ap), "l"(bp[j]), "l"(Z));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc[i][j]) : "l"(acc[i][j]), "l"(pr));
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const long long m = m0 + ty * 8 + i;
    if (m >= M) continue;
    float* row = out0 + b * M * N + m * N;
    const long long n = n0 + tx * TN;
    float v[TN];
#pragma unroll
    for (int j = 0; j < TN / 2; ++j) asm("mov.b64 {%0, %1}, %2;" : "=f"(v[2 * j]), "=f"(v[2 * j + 1]) : "l"(acc[i][j]));
#pragma unroll
    for (int h = 0; h < TN / 4; ++h)
      if (n + 4 * h < N) *reinterpret_cast<float4*>(row + n + 4 * h) = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
  }
}
)SFXDOT";

}  // namespace

KernelSource lower_dot(const Graph& g, const Program& p) {
  if (!dot_alone(g, p)) throw Error(SFX_ERR_INVALID, "not a matmul-only program");
  const int node = p.roots[0];
  const Node& n = g.nodes[node];
  if (n.op == SFX_OP_LIBRARY_CALL && n.kind != SFX_CALLEE_MATMUL)
    throw Error(SFX_ERR_EXEC, "library call 'opaque' is not executable");  // exec.cpp:209
  const Node& A = g.nodes[n.operands[0]];
  const int r = n.rank();
  const int64_t M = n.dims[r - 2], N = n.dims[r - 1], K = A.dims[r - 1];
  int64_t batch = 1;
  for (int i = 0; i < r - 2; ++i) batch *= n.dims[i];

  const bool f32 = n.dtype == SFX_F32;
  // packed-pair large-tile kernel: f32, both operands in memory, 16-byte rows
  const bool packed = f32 && M >= 128 && N >= 64 && K % 4 == 0 && N % 4 == 0 &&
                      !g.nodes[n.operands[0]].is_splat() && !g.nodes[n.operands[1]].is_splat() && dot_packed();
  int BM, BN, TM, TN;
  if (M >= 128 && N >= 128) BM = 128, BN = 128, TM = 8, TN = 8;
  else if (M >= 64 && N >= 64) BM = 64, BN = 64, TM = 4, TN = 4;
  else if (N <= 16) BM = 256, BN = 16, TM = 4, TN = 4;
  else BM = 32, BN = 32, TM = 2, TN = 2;
  const int64_t tiles_n = (N + BN - 1) / BN, tiles_m = (M + BM - 1) / BM;
  const int64_t grid = tiles_n * tiles_m * batch;
  if (grid >= (int64_t{1} << 31)) throw Error(SFX_ERR_UNSUPPORTED, "matmul " + n.id + " needs more than 2^31 CTAs");

  KernelSource ks;
  ks.strategy = "dot";
  std::string name;
  for (char ch : n.id) name += std::isalnum(static_cast<unsigned char>(ch)) ? ch : '_';
  if (name.size() > 40) name.resize(40);
  ks.entry = "sfx_dot_" + name;
  ks.inputs = p.inputs;
  ks.outputs = p.roots;
  ks.algorithmic_bytes = (n.numel() + A.numel() + g.nodes[n.operands[1]].numel()) * 4;
  ks.grid_x = grid;
  ks.block = (BM / TM) * (BN / TN);
  ks.smem = 0;
  ks.vector_width = 1;

  std::string params;
  std::map<int, std::string> ptr;
  for (size_t k = 0; k < p.inputs.size(); ++k) {
    ptr[p.inputs[k]] = "in" + std::to_string(k);
    params += std::string("const ") + ctype(g.nodes[p.inputs[k]].dtype) + "* __restrict__ in" + std::to_string(k) + ", ";
  }
  params += std::string(ctype(n.dtype)) + "* __restrict__ out0, unsigned* __restrict__ ws";
  if (packed) {
    // 128 x 128 tiles (8 x 8 per thread), or 128 x 64 (8 x 4) when N < 128
    const int PBN = N >= 128 ? 128 : 64, PTN = PBN / 16;
    const int64_t ptn = (N + PBN - 1) / PBN, ptm = (M + 127) / 128;
    ks.grid_x = ptn * ptm * batch;
    ks.smem = (3 * 128 * (32 + 4) + 3 * 32 * (PBN + 4)) * 4;
    std::string body2 = subst(kDotKernel2, {{"$TILES_N", fmt_i(ptn)},
                                            {"$TILES_M", fmt_i(ptm)},
                                            {"$BN", std::to_string(PBN)},
                                            {"$TN", std::to_string(PTN)},
                                            {"$ENTRY", ks.entry},
                                            {"$PARAMS", params},
                                            {"$A", ptr.at(n.operands[0])},
                                            {"$B", ptr.at(n.operands[1])},
                                            {"$M", fmt_i(M)},
                                            {"$N", fmt_i(N)},
                                            {"$K", fmt_i(K)}});
    ks.code = std::string(kPrelude) + "\n" + body2;
    std::ostringstream note;
    note << (p.barrier ? "matmul barrier [" : "matmul group [") << batch << " x " << M << " x " << K << "] @ [" << K
         << " x " << N << "]: tile 128x" << PBN << "x32, 8x" << PTN << " per thread, 3-stage cp.async pipeline, packed "
         << "fp32x2 products and sums, " << ks.grid_x << " CTAs; sequential-k fp32 (bit-exact)";
    ks.note = note.str();
    return ks;
  }
  std::string body = subst(kDotKernel, {{"$TILES_N", fmt_i(tiles_n)},
                                        {"$TILES_M", fmt_i(tiles_m)},
                                        {"$BM", std::to_string(BM)},
                                        {"$BN", std::to_string(BN)},
                                        {"$TM", std::to_string(TM)},
                                        {"$TN", std::to_string(TN)},
                                        {"$T4", f32 ? "float4" : "int4"},
                                        {"$T", f32 ? "float" : "int"},
                                        {"$ENTRY", ks.entry},
                                        {"$PARAMS", params},
                                        {"$M", fmt_i(M)},
                                        {"$N", fmt_i(N)},
                                        {"$K", fmt_i(K)}});
  // $LOAD_A(expr) -> __ldg(inK + (expr)), or the literal of a splat constant
  auto expand = [&](const std::string& key, int operand) {
    const Node& o = g.nodes[operand];
    size_t pos;
    while ((pos = body.find(key)) != std::string::npos) {
      size_t open = pos + key.size();  // at '('
      int depth = 0;
      size_t close = open;
      for (; close < body.size(); ++close) {
        if (body[close] == '(') ++depth;
        if (body[close] == ')' && --depth == 0) break;
      }
      std::string expr = body.substr(open + 1, close - open - 1);
      std::string rep;
      if (o.is_splat())
        rep = "T(" + (f32 ? fmt_f32(o.literal[0]) : fmt_i(static_cast<int32_t>(o.literal[0]))) + ")";
      else
        rep = "__ldg(" + ptr.at(operand) + " + (" + expr + "))";
      body.replace(pos, close + 1 - pos, rep);
    }
  };
  expand("$LOAD_A", n.operands[0]);
  expand("$LOAD_B", n.operands[1]);
  ks.code = std::string(kPrelude) + "\n" + body;
  std::ostringstream note;
  note << (p.barrier ? "matmul barrier [" : "matmul group [") << batch << " x " << M << " x " << K << "] @ [" << K << " x " << N << "]: tile " << BM
       << "x" << BN << "x16, " << TM << "x" << TN << " per thread, " << grid << " CTAs; sequential-k fp32 (bit-exact)";
  ks.note = note.str();
  return ks;
}

}  // namespace sfx
