// Device prelude prepended to every generated stitched kernel (compiled by
// NVRTC for sm_100a with -fmad=false, IEEE div/sqrt).  Scalar semantics follow
// the reference's compute_element / apply_unary / apply_binary exactly
// (reference proj/src/exec.cpp:18-65, 141-204):
//   max/min are std::max/std::min ((a<b)?b:a, (b<a)?b:a) — NaN handling differs
//   from fmaxf; compare yields 1/0; select tests pred != 0; scale multiplies in
//   double; rsqrt is 1/sqrt; i32 arithmetic wraps.
// Self-contained: no CUDA headers, so NVRTC needs no include path.
typedef unsigned int sfx_u32;
typedef unsigned long long sfx_u64;

struct __align__(16) sfx_f4 { float x, y, z, w; };
struct __align__(16) sfx_i4 { int x, y, z, w; };

// ---- f32 ----
__device__ __forceinline__ float sfx_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sfx_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float sfx_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float sfx_max(float a, float b) { return (a < b) ? b : a; }
__device__ __forceinline__ float sfx_min(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ float sfx_neg(float a) { return -a; }
__device__ __forceinline__ float sfx_cmp(float a, float b) { return a > b ? 1.0f : 0.0f; }
__device__ __forceinline__ float sfx_sel(float p, float t, float f) { return p != 0.0f ? t : f; }
__device__ __forceinline__ float sfx_scale_d(float a, double s) { return (float)((double)a * s); }
__device__ __forceinline__ float sfx_scale_f(float a, float s) { return __fmul_rn(a, s); }
// float(x * double(s)) in FP32: s = hi + lo with hi = s truncated to float and
// lo = float(s - hi) of the same sign; one rounding of a value within 2^-48
// relative of x*s.  Same float as the reference except at near-midpoints (1 ulp).
__device__ __forceinline__ float sfx_scale_2f(float a, float hi, float lo) {
  return __fmaf_rn(a, hi, __fmul_rn(a, lo));
}
__device__ __forceinline__ float sfx_exp(float a) { return expf(a); }
__device__ __forceinline__ float sfx_log(float a) { return logf(a); }
__device__ __forceinline__ float sfx_div(float a, float b) { return __fdiv_rn(a, b); }
// a / b for a divisor computed from a reduction (row / column constant): one
// IEEE reciprocal per divisor value, then a multiply (<= 1 ulp from a / b);
// zero, infinite, NaN or subnormal-range divisors take the IEEE division.
__device__ __forceinline__ float sfx_rcp(float b) { return __frcp_rn(b); }
__device__ __forceinline__ float sfx_div_rc(float a, float b, float r) {
  return (fabsf(b) > 0x1p-126f && fabsf(b) < 0x1p126f) ? __fmul_rn(a, r) : __fdiv_rn(a, b);
}
__device__ __forceinline__ float sfx_pow(float a, float b) { return powf(a, b); }
__device__ __forceinline__ float sfx_tanh(float a) { return tanhf(a); }
__device__ __forceinline__ float sfx_sqrt(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ float sfx_rsqrt(float a) { return __fdiv_rn(1.0f, __fsqrt_rn(a)); }

// ---- i32 (two's-complement wrap, like the reference's x86 build) ----
__device__ __forceinline__ int sfx_add(int a, int b) { return (int)((sfx_u32)a + (sfx_u32)b); }
__device__ __forceinline__ int sfx_sub(int a, int b) { return (int)((sfx_u32)a - (sfx_u32)b); }
__device__ __forceinline__ int sfx_mul(int a, int b) { return (int)((sfx_u32)a * (sfx_u32)b); }
__device__ __forceinline__ int sfx_max(int a, int b) { return (a < b) ? b : a; }
__device__ __forceinline__ int sfx_min(int a, int b) { return (b < a) ? b : a; }
// ptxas 12.9 for sm_100a miscompiles i32 max/min chains over negated values
// (it forms VIMNMX3 and drops one source's negation; found by the random-graph
// parity suite, device stream graph 157 — the PTX is correct).  Negating via a
// multiply by -1 held in constant memory keeps the negation out of ptxas'
// operand-modifier folding.
__constant__ int sfx_c_neg1 = -1;
__device__ __forceinline__ int sfx_neg(int a) { return (int)((sfx_u32)a * (sfx_u32)sfx_c_neg1); }
__device__ __forceinline__ int sfx_cmp(int a, int b) { return a > b ? 1 : 0; }
__device__ __forceinline__ int sfx_sel(int p, int t, int f) { return p != 0 ? t : f; }
// static_cast<int32_t>(x * scalar) on x86-64 (cvttsd2si): out-of-range/NaN -> INT_MIN
__device__ __forceinline__ int sfx_scale_d(int a, double s) {
  double p = (double)a * s;
  if (!(p > -2147483649.0 && p < 2147483648.0)) return (int)0x80000000u;
  return (int)p;
}

__device__ __forceinline__ float sfx_bits_f(int a) { return __int_as_float(a); }
__device__ __forceinline__ int sfx_bits_i(float a) { return __float_as_int(a); }

// ---- reduce folds (reference exec.cpp:67-74: sum = add, max/min = std::max/min) ----
__device__ __forceinline__ float sfx_fold_sum(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ int sfx_fold_sum(int a, int b) { return sfx_add(a, b); }
__device__ __forceinline__ double sfx_fold_sum(double a, float b) { return a + (double)b; }
__device__ __forceinline__ double sfx_fold_sum(double a, double b) { return a + b; }
// Parallel max/min: the sequential std::max fold returns the first element if
// it is NaN, else the max over the non-NaN elements.  Partial folds therefore
// ignore NaN (fmaxf/fminf semantics) and the first element is re-applied at the end.
__device__ __forceinline__ float sfx_fold_pmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float sfx_fold_pmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ int sfx_fold_pmax(int a, int b) { return a < b ? b : a; }
__device__ __forceinline__ int sfx_fold_pmin(int a, int b) { return b < a ? b : a; }
__device__ __forceinline__ float sfx_fold_first(float first, float acc) { return (first != first) ? first : acc; }
__device__ __forceinline__ int sfx_fold_first(int first, int acc) { return acc; }

// ---- memory ----
// Streaming 128-bit loads: read-only path, no L1 allocation (data read once).
// Not `volatile`: the inputs are read-only for the kernel's lifetime, and the
// scheduler must be free to hoist the next rows' loads above the current
// row's arithmetic (memory-level parallelism).
__device__ __forceinline__ sfx_f4 sfx_ld4s(const float* p) {
  sfx_f4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ sfx_i4 sfx_ld4s(const int* p) {
  sfx_i4 v;
  asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ sfx_f4 sfx_lds4(const float* p) { return *reinterpret_cast<const sfx_f4*>(p); }
__device__ __forceinline__ void sfx_sts4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<sfx_f4*>(p) = sfx_f4{a, b, c, d};
}

// ---- cross-rank flags in peer memory (column combine over NVLink) ----
__device__ __forceinline__ void sfx_st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned sfx_ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long sfx_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned sfx_ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Grid-wide barrier of a co-resident grid (one wave, cooperative launch):
// arrival counter ctr[0] grows by gridDim.x*gridDim.y per barrier; barrier k
// (1-based) waits for k*G arrivals.  sfx_grid_exit resets the counters once
// every CTA has passed its last barrier, so the next launch starts from zero.
__device__ __forceinline__ void sfx_grid_barrier(unsigned* ctr, unsigned k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = k * gridDim.x * gridDim.y;
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned long long t0 = sfx_globaltimer();
    while (sfx_ld_acquire_gpu(ctr) < target) {
      if (sfx_globaltimer() - t0 > 20000000000ull) __trap();
      __nanosleep(32);
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void sfx_grid_exit(unsigned* ctr) {
  if (threadIdx.x == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x * gridDim.y - 1u) {
    ctr[0] = 0u;
    ctr[1] = 0u;
  }
}
// Host-streaming gate: wait until the copy stream has published chunk count
// `need` (cuStreamWriteValue32 after the chunk's host->device copies).
__device__ __forceinline__ void sfx_gate_wait(const unsigned* gate, unsigned need) {
  const unsigned long long t0 = sfx_globaltimer();
  while (sfx_ld_acquire_sys(gate) < need) {
    if (sfx_globaltimer() - t0 > 20000000000ull) __trap();
    __nanosleep(128);
  }
}
// Wait until a peer has published sequence number `seq` (wrap-safe).  A rank
// that never arrives (crashed process, mismatched graphs) traps after 300 s
// instead of hanging the GPU; ranks legitimately drift apart by seconds (a
// first-use NVRTC compile on one rank, time-sliced ranks sharing a GPU).
__device__ __forceinline__ void sfx_peer_wait(const unsigned* flag, unsigned seq) {
  const unsigned long long t0 = sfx_globaltimer();
  while ((int)(sfx_ld_acquire_sys(flag) - seq) < 0) {
    if (sfx_globaltimer() - t0 > 300000000000ull) __trap();
    __nanosleep(64);
  }
}

// ---- TMA bulk copies + mbarrier (sm_90+/sm_100a), used by the pipelined row template ----
__device__ __forceinline__ unsigned sfx_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void sfx_mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sfx_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void sfx_fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void sfx_mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sfx_smem_u32(bar)), "r"(bytes)
               : "memory");
}
// one contiguous global -> shared copy by the TMA engine, completing on `bar`
__device__ __forceinline__ void sfx_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(sfx_smem_u32(dst)), "l"(src), "r"(bytes), "r"(sfx_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sfx_mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "SFX_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra SFX_DONE;\n"
      "bra SFX_WAIT;\n"
      "SFX_DONE:\n"
      "}\n" :: "r"(sfx_smem_u32(bar)), "r"(parity) : "memory");
}
// ---- thread-block clusters: distributed shared memory (long-row cluster template) ----
__device__ __forceinline__ unsigned sfx_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// every CTA of the cluster arrives (release) and waits (acquire): smem writes
// before it are visible to DSMEM reads after it, cluster-wide
__device__ __forceinline__ void sfx_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned sfx_dsmem_addr(const void* p, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(sfx_smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ float sfx_dsmem_ld(const float* p, unsigned rank) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(sfx_dsmem_addr(p, rank)) : "memory");
  return v;
}
__device__ __forceinline__ double sfx_dsmem_ld(const double* p, unsigned rank) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(sfx_dsmem_addr(p, rank)) : "memory");
  return v;
}
__device__ __forceinline__ int sfx_dsmem_ld(const int* p, unsigned rank) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(sfx_dsmem_addr(p, rank)) : "memory");
  return v;
}

// Cluster combine by push: st.async writes a partial into `rank`'s copy of `p`
// and completes that CTA's mbarrier transaction for its bytes, so a CTA waits
// on its own mbarrier for all of the cluster's partials — no cluster barrier
// (whose release / acquire is a GPU-scope MEMBAR + L1 invalidation) per
// reduction level.
__device__ __forceinline__ void sfx_dsmem_push(float* p, float v, unsigned long long* bar, unsigned rank) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
               :: "r"(sfx_dsmem_addr(p, rank)), "r"(__float_as_uint(v)), "r"(sfx_dsmem_addr(bar, rank)) : "memory");
}
__device__ __forceinline__ void sfx_dsmem_push(double* p, double v, unsigned long long* bar, unsigned rank) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
               :: "r"(sfx_dsmem_addr(p, rank)), "l"((unsigned long long)__double_as_longlong(v)),
                  "r"(sfx_dsmem_addr(bar, rank)) : "memory");
}
__device__ __forceinline__ void sfx_dsmem_push(int* p, int v, unsigned long long* bar, unsigned rank) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
               :: "r"(sfx_dsmem_addr(p, rank)), "r"(v), "r"(sfx_dsmem_addr(bar, rank)) : "memory");
}
// Per-thread asynchronous global -> shared copies (LDGSTS, L2 only): a thread
// reads back only what it copied itself, after cp.async.wait_group.
__device__ __forceinline__ void sfx_cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sfx_smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void sfx_cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void sfx_cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }
// split cluster barrier: a relaxed arrive (no memory ordering; the mbarrier
// inits are published by fence.mbarrier_init) and the matching wait
__device__ __forceinline__ void sfx_cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void sfx_cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// mbarrier phase wait that traps after 10 s instead of hanging the GPU
__device__ __forceinline__ void sfx_mbar_wait_bounded(unsigned long long* bar, unsigned parity) {
  const unsigned long long t0 = sfx_globaltimer();
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done) : "r"(sfx_smem_u32(bar)), "r"(parity) : "memory");
    if (!done && sfx_globaltimer() - t0 > 10000000000ull) __trap();
  }
}

// Reused 128-bit loads (broadcast vectors): default caching.
__device__ __forceinline__ sfx_f4 sfx_ld4(const float* p) { return *reinterpret_cast<const sfx_f4*>(p); }
__device__ __forceinline__ sfx_i4 sfx_ld4(const int* p) { return *reinterpret_cast<const sfx_i4*>(p); }
__device__ __forceinline__ float sfx_ld(const float* p) { return __ldg(p); }
__device__ __forceinline__ int sfx_ld(const int* p) { return __ldg(p); }
// Root stores: streaming (st.global.cs, evict-first in L2) — a root is written
// once and the inputs still streaming in keep the L2 (measured on B200:
// probs_d 463 -> 449 us, ctx_r 37.2 -> 35.3 us, h1 66.0 -> 63.9 us).
__device__ __forceinline__ void sfx_st4(float* p, float a, float b, float c, float d) {
#if defined(SFX_EXP_WB_STORES)  // A/B: default write-back stores
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
#elif defined(SFX_EXP_ST_NOCLOBBER)  // A/B: no compiler memory barrier at each store
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d));
#else
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
#endif
}
__device__ __forceinline__ void sfx_st4(int* p, int a, int b, int c, int d) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ---- cross-thread combine ----
__device__ __forceinline__ float sfx_shfl_xor(float v, int m, sfx_u32 mask) { return __shfl_xor_sync(mask, v, m); }
__device__ __forceinline__ int sfx_shfl_xor(int v, int m, sfx_u32 mask) { return __shfl_xor_sync(mask, v, m); }
__device__ __forceinline__ float sfx_shfl(float v, int src, sfx_u32 mask) { return __shfl_sync(mask, v, src); }
__device__ __forceinline__ int sfx_shfl(int v, int src, sfx_u32 mask) { return __shfl_sync(mask, v, src); }
