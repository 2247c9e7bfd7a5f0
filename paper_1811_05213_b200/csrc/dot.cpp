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
#include "lower_impl.hpp"

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
#define A_KFAST $A_KFAST
#define B_KFAST $B_KFAST
#define PACKED $PACKED
#define VEC $VEC
typedef $T T;
typedef $T4 T4;

extern "C" __global__ void __launch_bounds__(NT, NT >= 256 ? 2 : 1) $ENTRY($PARAMS) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const long long M = $M, N = $N, K = $K;
$PROLOGUE
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
#if VEC
  // stitched operands evaluated 4 elements at a time along their contiguous
  // axis (sfx_opA4 / sfx_opB4: 128-bit loads where the sources allow)
  float4 ra[LA / 4], rb[LB / 4];
  auto fetch = [&](long long k0) {
#pragma unroll
    for (int i = 0; i < LA / 4; ++i) {
      const int e = tid + i * NT;
      const int row = A_KFAST ? e / (BK / 4) : (e % (BM / 4)) * 4;
      const int kk = A_KFAST ? (e % (BK / 4)) * 4 : e / (BM / 4);
      const long long m = m0 + row, k = k0 + kk;
      ra[i] = (m < M && k < K) ? sfx_opA4(b, m, k) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < LB / 4; ++i) {
      const int e = tid + i * NT;
      const int kk = B_KFAST ? (e % (BK / 4)) * 4 : e / (BN / 4);
      const int col = B_KFAST ? e / (BK / 4) : (e % (BN / 4)) * 4;
      const long long k = k0 + kk, n = n0 + col;
      rb[i] = (k < K && n < N) ? sfx_opB4(b, k, n) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA / 4; ++i) {
      const int e = tid + i * NT;
      if (A_KFAST) {
        const int row = e / (BK / 4), kk = (e % (BK / 4)) * 4;
        As[buf][kk][row] = ra[i].x; As[buf][kk + 1][row] = ra[i].y;
        As[buf][kk + 2][row] = ra[i].z; As[buf][kk + 3][row] = ra[i].w;
      } else {
        *reinterpret_cast<float4*>(&As[buf][e / (BM / 4)][(e % (BM / 4)) * 4]) = ra[i];
      }
    }
#pragma unroll
    for (int i = 0; i < LB / 4; ++i) {
      const int e = tid + i * NT;
      if (B_KFAST) {
        const int col = e / (BK / 4), kk = (e % (BK / 4)) * 4;
        Bs[buf][kk][col] = rb[i].x; Bs[buf][kk + 1][col] = rb[i].y;
        Bs[buf][kk + 2][col] = rb[i].z; Bs[buf][kk + 3][col] = rb[i].w;
      } else {
        *reinterpret_cast<float4*>(&Bs[buf][e / (BN / 4)][(e % (BN / 4)) * 4]) = rb[i];
      }
    }
  };
#else
  T ra[LA], rb[LB];
  // staging order: consecutive threads take consecutive k (A_KFAST / B_KFAST)
  // or consecutive m / n, whichever is contiguous in the operand's source memory
#define A_ROW(e) (A_KFAST ? (e) / BK : (e) % BM)
#define A_KK(e) (A_KFAST ? (e) % BK : (e) / BM)
#define B_KK(e) (B_KFAST ? (e) % BK : (e) / BN)
#define B_COL(e) (B_KFAST ? (e) / BK : (e) % BN)
  auto fetch = [&](long long k0) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = tid + i * NT, row = A_ROW(e), kk = A_KK(e);
      const long long m = m0 + row, k = k0 + kk;
      ra[i] = (m < M && k < K) ? $LOAD_A(b * M * K + m * K + k) : T(0);
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = tid + i * NT, kk = B_KK(e), col = B_COL(e);
      const long long k = k0 + kk, n = n0 + col;
      rb[i] = (k < K && n < N) ? $LOAD_B(b * K * N + k * N + n) : T(0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = tid + i * NT;
      As[buf][A_KK(e)][A_ROW(e)] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = tid + i * NT;
      Bs[buf][B_KK(e)][B_COL(e)] = rb[i];
    }
  };
#endif
#if PACKED
  // f32 on the packed fp32x2 datapath (see kDotKernel2): t = fma(a, b, Z),
  // acc = acc + t, Z a zero ptxas cannot see
  typedef unsigned long long u64;
  unsigned dsz;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
  const float zf = __uint_as_float(dsz >> 20);
  u64 Z;
  asm("mov.b64 %0, {%1, %2};" : "=l"(Z) : "f"(zf), "f"(zf));
  u64 acc2[TM][TN / 2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN / 2; ++j) acc2[i][j] = 0ull;
#else
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);
#endif
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
#if PACKED
      u64 vp[TN / 2];
#pragma unroll
      for (int j = 0; j < TN / 2; ++j) asm("mov.b64 %0, {%1, %2};" : "=l"(vp[j]) : "f"(v[2 * j]), "f"(v[2 * j + 1]));
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        u64 ap;
        asm("mov.b64 %0, {%1, %2};" : "=l"(ap) : "f"(a[i]), "f"(a[i]));
#pragma unroll
        for (int j = 0; j < TN / 2; ++j) {
          u64 pr;
          asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pr) : "l"(ap), "l"(vp[j]), "l"(Z));
          asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc2[i][j]) : "l"(acc2[i][j]), "l"(pr));
        }
      }
#else
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = sfx_add(acc[i][j], sfx_mul(a[i], v[j]));
#endif
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
#if PACKED
    T accr[TN];
#pragma unroll
    for (int j = 0; j < TN / 2; ++j)
      asm("mov.b64 {%0, %1}, %2;" : "=f"(accr[2 * j]), "=f"(accr[2 * j + 1]) : "l"(acc2[i][j]));
#else
    const T* accr = acc[i];
#endif
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const long long n = n0 + tx * TN + j;
      if (n < N) row[n] = accr[j];
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
                                        {"$K", fmt_i(K)},
                                        {"$PROLOGUE", ""},
                                        {"$A_KFAST", "1"},
                                        {"$B_KFAST", "0"},
                                        {"$PACKED", f32 && TN % 2 == 0 && dot_packed() ? "1" : "0"},
                                        {"$VEC", "0"}});
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


// fuse_dot groups whose only root is the matmul and whose other members are
// elementwise / layout ops producing its operands (the reference planner with
// fuse_dot stitches e.g. bias add + head reshape + transpose into Q K^T, or the
// softmax normalisation x dropout mask into P V; fusion.cpp / span.cpp): the
// register-staged SIMT matmul above, with each operand element computed from the
// group's externals where the tile is staged (one generated expression per
// operand, the map template's index algebra) instead of read from a
// materialised tensor.  Same k order, same roundings: bit-identical to the
// reference's dot_loop over the stitched operands.
bool dot_prologue_ok(const Graph& g, const Program& p, std::string* why) {
  auto fail = [&](const std::string& w) {
    if (why) *why = w;
    return false;
  };
  int dot = -1;
  for (int m : p.members) {
    const Node& n = g.nodes[m];
    if (is_matmul(n)) {
      if (dot >= 0) return fail("more than one matmul");
      dot = m;
      continue;
    }
    switch (n.op) {
      case SFX_OP_ELEMENTWISE: case SFX_OP_RESHAPE: case SFX_OP_BITCAST: case SFX_OP_TRANSPOSE: case SFX_OP_BROADCAST:
        break;
      case SFX_OP_REDUCE:
        if (n.reduce_dims.empty() || n.numel() == g.nodes[n.operands[0]].numel()) break;
        return fail("a reduction feeds the matmul");
      default:
        return fail("unsupported member " + n.id);
    }
  }
  if (dot < 0) return fail("no matmul");
  if (p.roots.size() != 1 || p.roots[0] != dot) return fail("the matmul is not the only root");
  if (g.nodes[dot].op != SFX_OP_BATCH_MATMUL) return fail("library call");
  return true;
}

// Host-side index map of a stitched operand: follows layout members
// (reshape / bitcast / transpose / broadcast / degenerate reduce) and the
// first full-size operand of elementwise members down to an external, and
// returns that external's linear index for element `idx` of `node` (-1 if the
// chain ends in a splat or a smaller tensor).
int64_t source_index(const Graph& g, const Program& p, int node, std::vector<int64_t> idx) {
  for (int guard = 0; guard < 256; ++guard) {
    const Node& n = g.nodes[node];
    auto linear = [](const std::vector<int64_t>& d, const std::vector<int64_t>& i) {
      int64_t l = 0;
      for (size_t k = 0; k < d.size(); ++k) l = l * d[k] + i[k];
      return l;
    };
    auto delinear = [](const std::vector<int64_t>& d, int64_t l) {
      std::vector<int64_t> i(d.size());
      for (size_t k = d.size(); k-- > 0;) {
        i[k] = l % d[k];
        l /= d[k];
      }
      return i;
    };
    if (!p.is_member(node)) return n.is_splat() ? -1 : linear(n.dims, idx);
    if (n.operands.empty()) return -1;
    switch (n.op) {
      case SFX_OP_ELEMENTWISE: {
        int next = -1;
        for (int o : n.operands)
          if (g.nodes[o].numel() == n.numel() && !g.nodes[o].is_splat()) {
            next = o;
            break;
          }
        if (next < 0) return -1;
        node = next;
        break;
      }
      case SFX_OP_RESHAPE: case SFX_OP_BITCAST: case SFX_OP_REDUCE:  // (degenerate reduce: a reshape)
        idx = delinear(g.nodes[n.operands[0]].dims, linear(n.dims, idx));
        node = n.operands[0];
        break;
      case SFX_OP_TRANSPOSE: {  // out[i] = in[perm applied]: in index j = out index at perm^-1
        std::vector<int64_t> in(idx.size());
        for (size_t k = 0; k < n.perm.size(); ++k) in[n.perm[k]] = idx[k];
        idx = in;
        node = n.operands[0];
        break;
      }
      case SFX_OP_BROADCAST: {
        std::vector<int64_t> in;
        for (int64_t d : n.dim_map) in.push_back(idx[d]);
        idx = in;
        node = n.operands[0];
        break;
      }
      default:
        return -1;
    }
  }
  return -1;
}

// true: the operand's source is contiguous along the contraction axis k (stage
// k-fastest); false: along m / n.  A is [.., M, K] (k last), B [.., K, N].
bool k_contiguous(const Graph& g, const Program& p, int operand, bool is_a) {
  const Node& o = g.nodes[operand];
  const int r = o.rank();
  if (r < 2) return is_a;
  std::vector<int64_t> base(r, 0);
  const int kd = is_a ? r - 1 : r - 2, md = is_a ? r - 2 : r - 1;
  if (o.dims[kd] < 2 || o.dims[md] < 2) return is_a;
  std::vector<int64_t> pk = base, pm = base;
  pk[kd] = 1;
  pm[md] = 1;
  const int64_t s0 = source_index(g, p, operand, base), sk = source_index(g, p, operand, pk),
                sm = source_index(g, p, operand, pm);
  if (s0 < 0 || sk < 0 || sm < 0) return is_a;
  const int64_t dk = std::llabs(sk - s0), dm = std::llabs(sm - s0);
  return dk == 1 ? true : dm == 1 ? false : is_a;
}

KernelSource lower_dot_prologue(const Graph& g, const Program& p) {
  std::string why;
  if (!dot_prologue_ok(g, p, &why)) throw Error(SFX_ERR_UNSUPPORTED, "dot prologue: " + why);
  const int node = p.roots[0];
  const Node& n = g.nodes[node];
  const Node& A = g.nodes[n.operands[0]];
  const Node& Bn = g.nodes[n.operands[1]];
  const int r = n.rank();
  const int64_t M = n.dims[r - 2], N = n.dims[r - 1], K = A.dims[r - 1];
  int64_t batch = 1;
  for (int i = 0; i < r - 2; ++i) batch *= n.dims[i];
  int BM, BN, TM, TN;
  if (M >= 128 && N >= 128) BM = 128, BN = 128, TM = 8, TN = 8;
  else if (M >= 64 && N >= 64) BM = 64, BN = 64, TM = 4, TN = 4;
  else if (N <= 16) BM = 256, BN = 16, TM = 4, TN = 4;
  else BM = 32, BN = 32, TM = 2, TN = 2;
  const int64_t tiles_n = (N + BN - 1) / BN, tiles_m = (M + BM - 1) / BM;
  const int64_t grid = tiles_n * tiles_m * batch;
  if (grid >= (int64_t{1} << 31)) throw Error(SFX_ERR_UNSUPPORTED, "matmul " + n.id + " needs more than 2^31 CTAs");
  lw::Ctx c = lw::make_ctx(g, p);
  KernelSource ks;
  ks.strategy = "dot";
  ks.entry = "sfx_dotp_" + c.name.substr(0, 40);
  ks.inputs = p.inputs;
  ks.outputs = p.roots;
  int64_t bytes = n.numel() * 4;
  for (int e : p.inputs) bytes += g.nodes[e].numel() * 4;
  ks.algorithmic_bytes = bytes;
  ks.grid_x = grid;
  ks.block = (BM / TM) * (BN / TN);
  ks.smem = 0;
  ks.vector_width = 1;
  const bool f32 = n.dtype == SFX_F32;
  std::string params;
  Emitter em(g, p, 1, c.wide);
  em.rcp_reduced_divisors = false;  // no reductions in the group: plain IEEE division
  for (size_t k = 0; k < p.inputs.size(); ++k) {
    em.input_ptr[p.inputs[k]] = "in" + std::to_string(k);
    params += std::string("const ") + ctype(g.nodes[p.inputs[k]].dtype) + "* __restrict__ in" + std::to_string(k) + ", ";
  }
  params += std::string(ctype(n.dtype)) + "* __restrict__ out0, unsigned* __restrict__ ws";
  Code pro;
  em.code = &pro;
  pro.indent = 1;
  auto operand = [&](const char* fn, const Node& op, int opnode) {
    pro.line(std::string("auto ") + fn + " = [&](long long L) -> " + ctype(n.dtype) + " {");
    pro.indent++;
    em.push();
    const std::string L = c.wide ? "L" : "((int)L)";
    std::string v = em.value(opnode, em.from_linear(em.uni(L), op.dims));
    pro.line("return " + v + ";");
    em.pop();
    pro.indent--;
    pro.line("};");
  };
  operand("sfx_opA", A, n.operands[0]);
  operand("sfx_opB", Bn, n.operands[1]);
  // stage each operand along the axis its main source is contiguous in
  const bool a_kfast = k_contiguous(g, p, n.operands[0], true);
  const bool b_kfast = k_contiguous(g, p, n.operands[1], false);
  // 4-wide evaluation along the staging axis when its extents allow
  const int NTT = (BM / TM) * (BN / TN);
  const int LAe = BM * 16 / NTT, LBe = 16 * BN / NTT;
  const bool vec = f32 && LAe % 4 == 0 && LBe % 4 == 0 && (a_kfast ? K % 4 == 0 : M % 4 == 0) &&
                   (b_kfast ? K % 4 == 0 : N % 4 == 0) && (a_kfast ? 16 % 4 == 0 : BM % 4 == 0) && dot_packed();
  if (vec) {
    Emitter em4(g, p, 4, c.wide);
    em4.rcp_reduced_divisors = false;
    em4.input_ptr = em.input_ptr;
    em4.code = &pro;
    auto operand4 = [&](const char* fn, const Node& op, int opnode, bool vec_on_last) {
      // (pb, pi, pj): batch index, then the operand's last two coordinates;
      // the 4 lanes step the last coordinate (vec_on_last) or the one before
      pro.line(std::string("auto ") + fn + " = [&](long long pb, long long pi, long long pj) -> float4 {");
      pro.indent++;
      em4.push();
      const std::string cb = c.wide ? "pb" : "((int)pb)", ci = c.wide ? "pi" : "((int)pi)", cj = c.wide ? "pj" : "((int)pj)";
      std::vector<int64_t> bdims(op.dims.begin(), op.dims.end() - 2);
      std::vector<Ix> base = bdims.empty() ? std::vector<Ix>{} : em4.from_linear(em4.uni(cb), bdims);
      std::string v[4];
      for (int lane = 0; lane < 4; ++lane) {
        em4.lane = lane;
        std::vector<Ix> comps = base;
        comps.push_back(vec_on_last ? em4.uni(ci) : em4.lane_plus(ci));
        comps.push_back(vec_on_last ? em4.lane_plus(cj) : em4.uni(cj));
        v[lane] = em4.value(opnode, comps);
      }
      pro.line("return make_float4(" + v[0] + ", " + v[1] + ", " + v[2] + ", " + v[3] + ");");
      em4.pop();
      pro.indent--;
      pro.line("};");
    };
    operand4("sfx_opA4", A, n.operands[0], a_kfast);   // A [.., M, K]: k is last
    operand4("sfx_opB4", Bn, n.operands[1], !b_kfast);  // B [.., K, N]: n is last
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
                                        {"$K", fmt_i(K)},
                                        {"$PROLOGUE", pro.text},
                                        {"$A_KFAST", a_kfast ? "1" : "0"},
                                        {"$B_KFAST", b_kfast ? "1" : "0"},
                                        {"$PACKED", f32 && TN % 2 == 0 && dot_packed() ? "1" : "0"},
                                        {"$VEC", vec ? "1" : "0"},
                                        {"$LOAD_A(", "sfx_opA("},
                                        {"$LOAD_B(", "sfx_opB("}});
  ks.code = std::string(kPrelude) + "\n" + body;
  std::ostringstream note;
  note << "fuse_dot group [" << batch << " x " << M << " x " << K << "] @ [" << K << " x " << N
       << "] with " << (p.members.size() - 1) << " stitched operand member(s) computed where the tiles are staged: tile "
       << BM << "x" << BN << "x16, " << TM << "x" << TN << " per thread, " << grid
       << " CTAs; sequential-k fp32 (bit-exact)";
  ks.note = note.str();
  return ks;
}

}  // namespace sfx
