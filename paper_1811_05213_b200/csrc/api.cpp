// C ABI (include/sfx.h): context + device buffer manager, per-group kernels
// (run_program twin), whole-module executor (run_compiled twin) with CUDA-graph
// replay, and the NCCL all-reduce for batch-crossing column reductions.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no cost unless a profiler attaches

#include "dyn.hpp"
#include "ir.hpp"
#include "jit.hpp"
#include "lower.hpp"
#include "sfx.h"

namespace {

thread_local std::string g_last_error;

template <typename F>
sfx_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return SFX_OK;
  } catch (const sfx::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = std::string("internal: ") + e.what();
    return SFX_ERR_INVALID;
  }
}

}  // namespace

// ---- NCCL (dlopen'ed: the library is used only for the cross-GPU combine) ----
namespace {
typedef struct { char internal[SFX_NCCL_ID_BYTES]; } nccl_id_t;
typedef void* nccl_comm_t;
struct Nccl {
  int (*GetUniqueId)(nccl_id_t*) = nullptr;
  int (*CommInitRank)(nccl_comm_t*, int, nccl_id_t, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, CUstream) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
const Nccl& nccl() {
  static Nccl n;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = "libnccl.so.2 not available";
      return;
    }
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(h, "ncclAllReduce"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!n.GetUniqueId || !n.CommInitRank || !n.AllReduce) err = "libnccl missing symbols";
  });
  if (!err.empty()) throw sfx::Error(SFX_ERR_NCCL, err);
  return n;
}
void check_nccl(int r, const char* what) {
  if (r == 0) return;
  const Nccl& n = nccl();
  throw sfx::Error(SFX_ERR_NCCL, std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "error"));
}
}  // namespace

struct sfx_ctx {
  int device = 0;
  CUdevice dev = 0;
  CUcontext cu = nullptr;
  std::atomic<int64_t> launches{0};
  std::mutex mu;
  std::multimap<uint64_t, CUdeviceptr> pool;  // freed blocks by size (buffer manager)
  std::map<CUdeviceptr, uint64_t> live;
  nccl_comm_t comm = nullptr;
  // peer-memory group (sfx_peer_create / sfx_peer_open)
  CUdeviceptr peer_base = 0;       // this rank's symmetric arena
  uint64_t peer_bytes = 0, peer_used = 0;
  CUdeviceptr peer_table = 0;      // device array [pn] of every rank's arena, mapped here
  std::vector<CUdeviceptr> peer_opened;
  int pn = 0, prank = 0;

  void bind() const { sfx::check_cu(sfx::driver().cuCtxSetCurrent(cu), "cuCtxSetCurrent"); }

  CUdeviceptr alloc(uint64_t bytes) {
    bytes = std::max<uint64_t>(256, (bytes + 255) / 256 * 256);
    std::lock_guard<std::mutex> lock(mu);
    auto it = pool.find(bytes);
    CUdeviceptr p = 0;
    if (it != pool.end()) {
      p = it->second;
      pool.erase(it);
    } else {
      bind();
      sfx::check_cu(sfx::driver().cuMemAlloc(&p, bytes), "cuMemAlloc");
    }
    live[p] = bytes;
    return p;
  }
  void release(CUdeviceptr p) {
    std::lock_guard<std::mutex> lock(mu);
    auto it = live.find(p);
    if (it == live.end()) throw sfx::Error(SFX_ERR_INVALID, "sfx_free of a pointer not from sfx_alloc");
    pool.emplace(it->second, p);
    live.erase(it);
  }
};

struct sfx_kernel {
  sfx_ctx* ctx = nullptr;
  sfx::KernelSource src;
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  // Workspace (cross-CTA tickets / partials; the kernels reset their tickets
  // on exit).  Launches on one stream are ordered, so each stream gets its own
  // workspace and launches on different streams never share one; `ws` is the
  // kernel's default (cross-rank kernels, whose launches are ordered on every
  // rank anyway, and launches captured outside sfx_graph_run).
  CUdeviceptr ws = 0;
  std::mutex ws_mu;
  std::map<CUstream, CUdeviceptr> stream_ws;
  uint64_t peer_off = 0;  // this kernel's region of the symmetric peer arena
  int regs = 0;
  int debug = 0;                    // sfx_compile_opts.debug_checks
  std::vector<int64_t> out_elems;   // per output slot (coverage check)
  std::string cubin_path;
};

// host streaming: per kernel gate[kMaxChunks] (set to 1 when chunk j's inputs
// landed) then done[kMaxChunks] (CTAs of chunk j that stored their rows)
constexpr int kMaxChunks = 64;
constexpr int kFlagWords = 2 * kMaxChunks;

// Streamed bytes per chunk on the host path (0 = the default policy below;
// SFX_HOST_CHUNK_BYTES overrides it, e.g. to exercise many chunks on small
// graphs in tests).
// Concurrent branches for independent groups in sfx_graph_run (SFX_GRAPH_BRANCHES=0
// turns them off, for A/B measurement).
constexpr int kBranches = 4;
bool graph_branches() {
  static const bool v = [] {
    const char* e = std::getenv("SFX_GRAPH_BRANCHES");
    return !(e && e[0] == '0');
  }();
  return v;
}

// SFX_HOST_STREAM=0 turns the chunk-streamed host path off (whole copies
// ordered by events; for A/B measurement).
bool host_streaming() {
  static const bool v = [] {
    const char* e = std::getenv("SFX_HOST_STREAM");
    return !(e && e[0] == '0');
  }();
  return v;
}

uint64_t host_chunk_bytes() {
  static const uint64_t v = [] {
    const char* e = std::getenv("SFX_HOST_CHUNK_BYTES");
    long long x = e ? std::atoll(e) : 0;
    return x > 0 ? static_cast<uint64_t>(x) : uint64_t{0};
  }();
  return v;
}

struct sfx_graph {
  sfx_ctx* ctx = nullptr;
  std::mutex run_mu;                 // one host thread enqueues at a time
  // CUDA-graph replays: every captured pointer set owns its kernels'
  // workspaces (replays of one exec are serialised by CUDA; different execs may
  // run concurrently on different streams)
  std::map<std::vector<uint64_t>, std::vector<CUdeviceptr>> captured_ws;
  sfx::Graph graph;
  std::vector<sfx_kernel*> kernels;  // per program: planned groups, then matmul barriers
  // host path: row / map kernels recompiled with the host-streaming gate code
  // (opts.host_stream), built on the first sfx_graph_run_host; null = use kernels[p]
  std::vector<sfx_kernel*> host_kernels;
  sfx_compile_opts opts{};
  int n_planned = 0;                 // programs that came from the CompileReport
  std::vector<int> order;            // program launch order (condensation Kahn order)
  std::vector<int> params;           // Parameter nodes, ascending id = param slot order
  std::map<int, CUdeviceptr> owned;  // dense constants and splat outputs (device-resident)
  // Intermediates (group roots that are not graph outputs, consumed by later
  // groups) are per launch context, like the workspaces: one set per stream for
  // eager runs (key {0, stream}) and one per captured pointer set (key {1,
  // params..., outputs...}), so concurrent runs on different streams never
  // share an intermediate buffer.  `last_mid[stream]` = the set the latest run
  // on that stream wrote (what sfx_graph_fetch reads).
  std::vector<int> mid_nodes;
  std::map<std::vector<uint64_t>, std::map<int, CUdeviceptr>> mids;
  std::map<CUstream, const std::map<int, CUdeviceptr>*> last_mid;
  std::map<std::vector<uint64_t>, std::pair<CUgraph, CUgraphExec>> captured;
  // Host path staging: two slots (params then outputs, plus the chunk flags),
  // used alternately, so run i+1's host->device copies land in one slot while
  // run i's kernels and copies back still use the other.  A slot is reused once
  // every stream of its previous run is past its last use (free_ev).
  struct HostSlot {
    std::vector<CUdeviceptr> bufs;
    CUdeviceptr flags = 0;          // per kernel: gate[kMaxChunks] + done[kMaxChunks]
    CUevent free_ev = nullptr;
    bool used = false;
  };
  HostSlot hslot[2];
  int hnext = 0;
  CUstream d2h = nullptr;              // host path: device->host copies overlap the next groups
  CUstream h2d = nullptr, h2d2 = nullptr;  // host path: host->device copies (chunks alternate)
  CUstream d2h2 = nullptr;                 // second device->host stream (chunks alternate)
  std::vector<CUstream> branch_streams;  // device path: independent groups run concurrently
  std::vector<CUevent> branch_events;    // per kernel completion, then fork / join
  std::vector<CUevent> events;
  CUevent join_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // host path: copy streams -> `s`
  std::vector<int> host_order;
};

namespace {

sfx_kernel* build_kernel(sfx_ctx* ctx, const sfx::Graph& g, int pi, const sfx_compile_opts* opts) {
  sfx_compile_opts o{};
  if (opts) o = *opts;
  auto k = std::make_unique<sfx_kernel>();
  k->ctx = ctx;
  k->src = sfx::lower_program(g, pi, o);
  k->debug = o.debug_checks;
  for (int r : k->src.outputs) k->out_elems.push_back(g.nodes[r].numel());
  sfx::Cubin cb = sfx::compile_cubin(k->src.code, k->src.entry, k->src.nvrtc_options);
  k->cubin_path = cb.path;
  ctx->bind();
  const sfx::Driver& d = sfx::driver();
  sfx::check_cu(d.cuModuleLoadData(&k->mod, cb.image.data()), "cuModuleLoadData");
  sfx::check_cu(d.cuModuleGetFunction(&k->fn, k->mod, k->src.entry.c_str()), "cuModuleGetFunction");
  d.cuFuncGetAttribute(&k->regs, CU_FUNC_ATTRIBUTE_NUM_REGS, k->fn);
  if (k->src.cluster > 8)
    sfx::check_cu(d.cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_NON_PORTABLE_CLUSTER_SIZE_ALLOWED, 1),
                  "cuFuncSetAttribute(non-portable cluster)");
  int static_smem = 0;
  d.cuFuncGetAttribute(&static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, k->fn);
  if (k->src.smem + static_smem > 48 * 1024)  // the 48 KB default bounds static + dynamic
    sfx::check_cu(d.cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, k->src.smem),
                  "cuFuncSetAttribute(smem)");
  if (k->src.peer_bytes > 0) {
    // regions are handed out in build order, identical on every rank
    if (!ctx->peer_table)
      throw sfx::Error(SFX_ERR_INVALID, "cross_rank kernel " + k->src.entry + " needs sfx_peer_open first");
    if (ctx->peer_used + static_cast<uint64_t>(k->src.peer_bytes) > ctx->peer_bytes)
      throw sfx::Error(SFX_ERR_INVALID, "peer arena too small: " + std::to_string(ctx->peer_bytes) + " bytes, need " +
                                            std::to_string(ctx->peer_used + k->src.peer_bytes));
    k->peer_off = ctx->peer_used;
    ctx->peer_used += static_cast<uint64_t>(k->src.peer_bytes);
  }
  if (k->src.workspace_bytes > 0) {
    k->ws = ctx->alloc(static_cast<uint64_t>(k->src.workspace_bytes));
    sfx::check_cu(d.cuMemsetD32Async(k->ws, 0, (k->src.workspace_bytes + 3) / 4, nullptr), "cuMemsetD32Async");
    sfx::check_cu(d.cuStreamSynchronize(nullptr), "cuStreamSynchronize");
  }
  return k.release();
}

// Host-streaming arguments of one launch (KernelSource::stream_R): null gate =
// no streaming, the kernel runs on resident inputs as usual.
struct StreamArgs {
  CUdeviceptr gate = 0, done = 0;
  long long chunk_elems = 0;
};

// Per-group launch log (metrics): SFX_LAUNCH_LOG=stderr|<path> writes
// one line per launch — kernel, template, grid / block / dynamic smem /
// registers, algorithmic bytes — and, outside stream capture, the launch's
// device time from CUDA events around it (the log synchronises every launch:
// a diagnostic mode, not for benchmarking), its GB/s and the fraction of
// SFX_PEAK_GBS (default 6538.6 GB/s, the measured B200 copy peak).  Launches
// recorded into a CUDA graph are logged as "captured", untimed.
struct LaunchLog {
  FILE* f = nullptr;
  double peak = 6538.6;
  std::mutex mu;
};
LaunchLog* launch_log() {
  static LaunchLog* log = []() -> LaunchLog* {
    const char* e = std::getenv("SFX_LAUNCH_LOG");
    if (!e || !e[0]) return nullptr;
    auto* L = new LaunchLog;
    L->f = std::strcmp(e, "stderr") == 0 ? stderr : std::fopen(e, "a");
    if (!L->f) {
      delete L;
      return nullptr;
    }
    if (const char* pk = std::getenv("SFX_PEAK_GBS")) L->peak = std::atof(pk) > 0 ? std::atof(pk) : L->peak;
    return L;
  }();
  return log;
}

void launch_raw(sfx_kernel* k, const std::vector<CUdeviceptr>& in, const std::vector<CUdeviceptr>& out, CUstream s,
                const StreamArgs& sa, bool drop_last_cta);

// One launch of a group's kernel.  With debug_checks, the coverage check of
// the reference's executor (exec.cpp:393-410: every root element written
// exactly once, "incomplete coverage" otherwise) runs around it.
void launch(sfx_kernel* k, const std::vector<CUdeviceptr>& in, const std::vector<CUdeviceptr>& out, CUstream s,
            const StreamArgs& sa = StreamArgs()) {
  if (!k->debug || sa.gate) {
    launch_raw(k, in, out, s, sa, false);
    return;
  }
  const sfx::Driver& d = sfx::driver();
  CUstreamCaptureStatus cap = CU_STREAM_CAPTURE_STATUS_NONE;
  sfx::check_cu(d.cuStreamIsCapturing(s, &cap), "cuStreamIsCapturing");
  if (cap != CU_STREAM_CAPTURE_STATUS_NONE)
    throw sfx::Error(SFX_ERR_INVALID, "debug_checks cannot run inside CUDA-graph capture");
  // canary A; elements still equal to it are re-checked with canary B (a value
  // the kernel legitimately computes cannot equal both)
  const uint32_t canary[2] = {0x7fa5a5a5u, 0xffc3c3c3u};
  std::vector<std::vector<uint32_t>> suspect(out.size());
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t i = 0; i < out.size(); ++i)
      sfx::check_cu(d.cuMemsetD32Async(out[i], canary[pass], k->out_elems[i], s), "cuMemsetD32Async");
    launch_raw(k, in, out, s, sa, k->debug == 2);
    sfx::check_cu(d.cuStreamSynchronize(s), "cuStreamSynchronize");
    bool any = false;
    for (size_t i = 0; i < out.size(); ++i) {
      std::vector<uint32_t> host(k->out_elems[i]);
      sfx::check_cu(d.cuMemcpyDtoH(host.data(), out[i], host.size() * 4), "cuMemcpyDtoH");
      std::vector<uint32_t> still;
      if (pass == 0) {
        for (size_t e = 0; e < host.size(); ++e)
          if (host[e] == canary[0]) still.push_back(static_cast<uint32_t>(e));
      } else {
        for (uint32_t e : suspect[i])
          if (host[e] == canary[1]) still.push_back(e);
      }
      suspect[i] = still;
      any = any || !still.empty();
    }
    if (!any) return;
  }
  for (size_t i = 0; i < out.size(); ++i)
    if (!suspect[i].empty())
      throw sfx::Error(SFX_ERR_EXEC, "incomplete coverage: " + k->src.entry + " left " +
                                         std::to_string(suspect[i].size()) + " element(s) of output " +
                                         std::to_string(i) + " unwritten (first: " + std::to_string(suspect[i][0]) +
                                         ")");
}

// Workspaces prepared for a capture in progress on this thread (sfx_graph_run),
// by kernel; null outside one.
thread_local const std::map<const sfx_kernel*, CUdeviceptr>* t_capture_ws = nullptr;

CUdeviceptr workspace_for(sfx_kernel* k, CUstream s) {
  if (k->src.workspace_bytes <= 0) return 0;
  if (t_capture_ws) {
    auto it = t_capture_ws->find(k);
    if (it != t_capture_ws->end()) return it->second;
  }
  if (k->src.peer_bytes > 0) return k->ws;  // cross-rank: one ordered sequence per rank
  const sfx::Driver& d = sfx::driver();
  CUstreamCaptureStatus cap = CU_STREAM_CAPTURE_STATUS_NONE;
  sfx::check_cu(d.cuStreamIsCapturing(s, &cap), "cuStreamIsCapturing");
  if (cap != CU_STREAM_CAPTURE_STATUS_NONE) return k->ws;  // captured by the caller: no allocation allowed
  std::lock_guard<std::mutex> lock(k->ws_mu);
  auto it = k->stream_ws.find(s);
  if (it != k->stream_ws.end()) return it->second;
  CUdeviceptr w = k->ctx->alloc(static_cast<uint64_t>(k->src.workspace_bytes));
  // zeroed in stream order, ahead of this stream's first launch
  sfx::check_cu(d.cuMemsetD32Async(w, 0, (k->src.workspace_bytes + 3) / 4, s), "cuMemsetD32Async");
  k->stream_ws.emplace(s, w);
  return w;
}

void launch_raw(sfx_kernel* k, const std::vector<CUdeviceptr>& in, const std::vector<CUdeviceptr>& out, CUstream s,
                const StreamArgs& sa, bool drop_last_cta) {
  if (in.size() != k->src.inputs.size())
    throw sfx::Error(SFX_ERR_INVALID, "expected " + std::to_string(k->src.inputs.size()) + " inputs");
  if (out.size() != k->src.outputs.size())
    throw sfx::Error(SFX_ERR_INVALID, "expected " + std::to_string(k->src.outputs.size()) + " outputs");
  std::vector<CUdeviceptr> vals;
  vals.reserve(in.size() + out.size() + 1);
  // every template assumes 16-byte aligned bases (128-bit ld/st, sfx_st4, TMA
  // bulk copies); a misaligned base (e.g. a tensor view at an odd offset) would
  // fault and poison the context, so it is refused here instead
  for (CUdeviceptr p : in) {
    if (!p) throw sfx::Error(SFX_ERR_EXEC, "null input pointer");
    if (p & 15) throw sfx::Error(SFX_ERR_INVALID, "input pointer not 16-byte aligned (" + k->src.entry + ")");
    vals.push_back(p);
  }
  for (CUdeviceptr p : out) {
    if (!p) throw sfx::Error(SFX_ERR_EXEC, "null output pointer");
    if (p & 15) throw sfx::Error(SFX_ERR_INVALID, "output pointer not 16-byte aligned (" + k->src.entry + ")");
    vals.push_back(p);
  }
  vals.push_back(workspace_for(k, s));
  std::vector<void*> args(vals.size());
  for (size_t i = 0; i < vals.size(); ++i) args[i] = &vals[i];
  CUdeviceptr peers = k->ctx->peer_table;
  unsigned long long poff = k->peer_off;
  int prank = k->ctx->prank, pn = k->ctx->pn;
  if (k->src.peer_bytes > 0) {
    args.push_back(&peers);
    args.push_back(&poff);
    args.push_back(&prank);
    args.push_back(&pn);
  }
  CUdeviceptr sgate = sa.gate, sdone = sa.done;
  long long schunk = sa.chunk_elems;
  if (k->src.stream_R > 0) {
    args.push_back(&sgate);
    args.push_back(&sdone);
    args.push_back(&schunk);
  } else if (sa.gate) {
    throw sfx::Error(SFX_ERR_INVALID, "internal: stream gate for a non-streaming kernel");
  }
  // programmatic dependent launch (every generated kernel begins with
  // griddepcontrol.wait, so stream order is preserved)
  CUlaunchAttribute attr[2];
  attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  attr[0].value.programmaticStreamSerializationAllowed = 1;
  unsigned n_attr = 1;
  if (k->src.cooperative) {  // grid barriers: the driver refuses a grid that cannot be co-resident
    attr[1].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
    attr[1].value.cooperative = 1;
    n_attr = 2;
  }
  CUlaunchConfig cfg{};
  cfg.gridDimX = static_cast<unsigned>(k->src.grid_x);
  cfg.gridDimY = static_cast<unsigned>(k->src.grid_y);
  if (drop_last_cta) {  // debug_checks=2 test hook
    if (cfg.gridDimY > 1) --cfg.gridDimY;
    else if (cfg.gridDimX > 1) --cfg.gridDimX;
  }
  cfg.gridDimZ = 1;
  cfg.blockDimX = static_cast<unsigned>(k->src.block);
  cfg.blockDimY = 1;
  cfg.blockDimZ = 1;
  cfg.sharedMemBytes = static_cast<unsigned>(k->src.smem);
  cfg.hStream = s;
  cfg.attrs = attr;
  cfg.numAttrs = n_attr;
  // one NVTX range per group launch, named by its kernel (ncu --nvtx / nsys timelines)
  nvtxRangePushA(k->src.entry.c_str());
  LaunchLog* log = launch_log();
  CUevent ev[2] = {nullptr, nullptr};
  if (log) {
    CUstreamCaptureStatus cs = CU_STREAM_CAPTURE_STATUS_NONE;
    sfx::driver().cuStreamIsCapturing(s, &cs);
    if (cs == CU_STREAM_CAPTURE_STATUS_NONE) {
      sfx::driver().cuEventCreate(&ev[0], CU_EVENT_DEFAULT);
      sfx::driver().cuEventCreate(&ev[1], CU_EVENT_DEFAULT);
      sfx::driver().cuEventRecord(ev[0], s);
    }
  }
  CUresult lr = sfx::driver().cuLaunchKernelEx(&cfg, k->fn, args.data(), nullptr);
  nvtxRangePop();
  if (log) {
    float ms = -1.0f;
    if (ev[0]) {
      sfx::driver().cuEventRecord(ev[1], s);
      if (lr == CUDA_SUCCESS && sfx::driver().cuEventSynchronize(ev[1]) == CUDA_SUCCESS)
        sfx::driver().cuEventElapsedTime(&ms, ev[0], ev[1]);
      sfx::driver().cuEventDestroy(ev[0]);
      sfx::driver().cuEventDestroy(ev[1]);
    }
    std::lock_guard<std::mutex> g(log->mu);
    std::fprintf(log->f, "sfx launch %s strategy=%s grid=%ux%u block=%u smem=%d regs=%d bytes=%lld", k->src.entry.c_str(),
                 k->src.strategy.c_str(), cfg.gridDimX, cfg.gridDimY, cfg.blockDimX, k->src.smem, k->regs,
                 static_cast<long long>(k->src.algorithmic_bytes));
    if (ms > 0.0f) {
      const double gbs = static_cast<double>(k->src.algorithmic_bytes) / (ms * 1e-3) / 1e9;
      std::fprintf(log->f, " us=%.2f GB/s=%.0f peak_frac=%.3f\n", ms * 1e3, gbs, gbs / log->peak);
    } else {
      std::fprintf(log->f, " %s\n", ev[0] ? "untimed" : "captured");
    }
    std::fflush(log->f);
  }
  sfx::check_cu(lr, "cuLaunchKernelEx");
  k->ctx->launches.fetch_add(1);
}

void destroy_kernel(sfx_kernel* k) {
  if (!k) return;
  try {
    k->ctx->bind();
    if (k->mod) sfx::driver().cuModuleUnload(k->mod);
    if (k->ws) k->ctx->release(k->ws);
    for (auto& [st, w] : k->stream_ws) k->ctx->release(w);
  } catch (...) {
  }
  delete k;
}

// Unfused instructions (fusion.cpp:259-263): the fusion barriers and any
// instruction no group took; run_compiled evaluates each densely
// (pipeline.cpp:124-127).  Each becomes one kernel, appended after the planned
// groups in instruction order.
void add_barrier_programs(sfx::Graph& g) {
  std::vector<bool> in_group(g.nodes.size(), false);
  for (const sfx::Program& p : g.programs)
    for (int m : p.members) in_group[m] = true;
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    const sfx::Node& n = g.nodes[i];
    if (in_group[i] || n.op == SFX_OP_PARAMETER || n.op == SFX_OP_CONSTANT) continue;
    if (n.op == SFX_OP_LIBRARY_CALL && n.kind != SFX_CALLEE_MATMUL)
      throw sfx::Error(SFX_ERR_EXEC, "library call 'opaque' is not executable");  // exec.cpp:209
    g.programs.push_back(sfx::barrier_program(g, static_cast<int>(i)));
  }
}

// run_compiled's condensation order (reference pipeline.cpp:67-131): one node
// per program plus one per remaining instruction, Kahn with sorted ready set.
std::vector<int> condensation_order(const sfx::Graph& g) {
  const int P = static_cast<int>(g.programs.size());
  std::vector<int> node_of(g.nodes.size(), -1);
  for (int p = 0; p < P; ++p)
    for (int m : g.programs[p].members) node_of[m] = p;
  int n = P;
  std::vector<int> singles;
  for (size_t i = 0; i < g.nodes.size(); ++i)
    if (node_of[i] < 0) {
      node_of[i] = n++;
      singles.push_back(static_cast<int>(i));
    }
  std::vector<std::set<int>> succ(n);
  std::vector<int> indeg(n, 0);
  for (size_t i = 0; i < g.nodes.size(); ++i)
    for (int op : g.nodes[i].operands) {
      int a = node_of[op], b = node_of[i];
      if (a != b && succ[a].insert(b).second) ++indeg[b];
    }
  std::vector<int> ready;
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) ready.push_back(i);
  std::vector<int> order;
  int processed = 0;
  while (!ready.empty()) {
    int v = ready.front();
    ready.erase(ready.begin());
    ++processed;
    if (v < P) order.push_back(v);
    for (int s : succ[v])
      if (--indeg[s] == 0) ready.insert(std::lower_bound(ready.begin(), ready.end(), s), s);
  }
  if (processed != n) throw sfx::Error(SFX_ERR_EXEC, "condensation is cyclic");
  return order;
}

// Launch order for the host-buffer path: any order respecting the groups'
// dataflow gives identical values; groups returning the most bytes go first so
// their device->host copies overlap the remaining host->device traffic.
std::vector<int> host_order(const sfx_graph* G) {
  const sfx::Graph& g = G->graph;
  const int P = static_cast<int>(g.programs.size());
  std::map<int, int> producer;
  for (int p = 0; p < P; ++p)
    for (int r : g.programs[p].roots) producer[r] = p;
  std::set<int> outs(g.outputs.begin(), g.outputs.end());
  std::vector<int64_t> d2h(P, 0);
  std::vector<std::set<int>> succ(P);
  std::vector<int> indeg(P, 0);
  for (int p = 0; p < P; ++p) {
    for (int r : g.programs[p].roots)
      if (outs.count(r)) d2h[p] += g.nodes[r].numel() * 4;
    for (int in : g.programs[p].inputs) {
      auto it = producer.find(in);
      if (it != producer.end() && it->second != p && succ[it->second].insert(p).second) ++indeg[p];
    }
  }
  std::vector<int> order, ready;
  for (int p = 0; p < P; ++p)
    if (!indeg[p]) ready.push_back(p);
  while (!ready.empty()) {
    auto best = std::min_element(ready.begin(), ready.end(), [&](int a, int b) {
      return d2h[a] != d2h[b] ? d2h[a] > d2h[b] : a < b;
    });
    int p = *best;
    ready.erase(best);
    order.push_back(p);
    for (int q : succ[p])
      if (--indeg[q] == 0) ready.push_back(q);
  }
  if (static_cast<int>(order.size()) != P) throw sfx::Error(SFX_ERR_EXEC, "group dependencies are cyclic");
  return order;
}

std::vector<CUdeviceptr> gather_ptrs(const sfx_graph* G, const std::vector<int>& nodes,
                                     const std::map<int, CUdeviceptr>& where) {
  std::vector<CUdeviceptr> v;
  for (int n : nodes) {
    auto it = where.find(n);
    if (it == where.end()) throw sfx::Error(SFX_ERR_EXEC, "missing external value " + G->graph.nodes[n].id);
    v.push_back(it->second);
  }
  return v;
}

// The intermediate set of launch context `key` (allocated on first use).
const std::map<int, CUdeviceptr>& mids_for(sfx_graph* G, const std::vector<uint64_t>& key) {
  auto it = G->mids.find(key);
  if (it != G->mids.end()) return it->second;
  std::map<int, CUdeviceptr>& m = G->mids[key];
  for (int r : G->mid_nodes) m[r] = G->ctx->alloc(G->graph.nodes[r].numel() * 4);
  return m;
}

std::vector<uint64_t> eager_key(CUstream s) { return {0, reinterpret_cast<uint64_t>(s)}; }

void graph_enqueue(sfx_graph* G, const uint64_t* params, const uint64_t* outputs, CUstream s,
                   const std::map<int, CUdeviceptr>& mid) {
  std::map<int, CUdeviceptr> where = G->owned;
  where.insert(mid.begin(), mid.end());
  G->last_mid[s] = &mid;
  for (size_t i = 0; i < G->params.size(); ++i) where[G->params[i]] = params[i];
  for (size_t i = 0; i < G->graph.outputs.size(); ++i) where[G->graph.outputs[i]] = outputs[i];
  const sfx::Driver& d = sfx::driver();
  for (size_t i = 0; i < G->graph.outputs.size(); ++i) {
    int o = G->graph.outputs[i];
    const sfx::Node& n = G->graph.nodes[o];
    if (n.op == SFX_OP_PARAMETER || n.op == SFX_OP_CONSTANT) {  // output with no producing group
      auto src = G->owned.count(o) ? G->owned.at(o) : where.at(o);
      for (size_t k = 0; k < G->params.size(); ++k)
        if (G->params[k] == o) src = params[k];
      if (src != outputs[i])
        sfx::check_cu(d.cuMemcpyDtoDAsync(outputs[i], src, n.numel() * 4, s), "cuMemcpyDtoDAsync");
    }
  }
  if (!graph_branches() || G->order.size() < 2) {
    for (int p : G->order) {
      sfx_kernel* k = G->kernels[p];
      launch(k, gather_ptrs(G, k->src.inputs, where), gather_ptrs(G, k->src.outputs, where), s);
    }
    return;
  }
  // Independent groups on parallel branches (fork/join with events; captured
  // as parallel CUDA-graph nodes), so one group's ramp and tail overlap
  // another's body instead of leaving HBM idle between launches.  Edges are
  // the groups' data dependencies (a group reads roots of earlier groups);
  // roots, workspaces and inputs are otherwise disjoint, so nothing else orders
  // them.  Within a branch, launches stay PDL-chained.
  const int K = static_cast<int>(G->kernels.size());
  if (G->branch_streams.empty()) {
    G->branch_streams.resize(kBranches - 1, nullptr);
    for (CUstream& st : G->branch_streams)
      sfx::check_cu(d.cuStreamCreate(&st, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    G->branch_events.resize(K + kBranches, nullptr);
    for (CUevent& e : G->branch_events) sfx::check_cu(d.cuEventCreate(&e, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  }
  std::map<int, int> producer;
  for (int p = 0; p < K; ++p)
    for (int r : G->kernels[p]->src.outputs) producer[r] = p;
  std::vector<CUstream> streams{s};
  streams.insert(streams.end(), G->branch_streams.begin(), G->branch_streams.end());
  std::vector<bool> forked(streams.size(), false);
  forked[0] = true;
  CUevent ev_fork = G->branch_events[K];
  sfx::check_cu(d.cuEventRecord(ev_fork, s), "cuEventRecord");
  std::vector<int> stream_of(K, -1);
  int next = 0, last_peer = -1;
  for (int p : G->order) {
    sfx_kernel* k = G->kernels[p];
    std::set<int> deps;
    for (int in : k->src.inputs) {
      auto it = producer.find(in);
      if (it != producer.end() && it->second != p) deps.insert(it->second);
    }
    // Kernels that exchange data with the other ranks (peer_bytes > 0) wait on
    // peers' kernels, so every rank must run them in the same order, one at a
    // time: each is chained after the previous one (condensation order, the
    // same on every rank).  On parallel branches rank A could run X while
    // rank B runs Y, each spinning on a peer kernel that cannot become resident.
    if (k->src.peer_bytes > 0) {
      if (last_peer >= 0) deps.insert(last_peer);
      last_peer = p;
    }
    int si;
    if (deps.empty()) {
      si = next;
      next = (next + 1) % static_cast<int>(streams.size());
    } else {
      si = stream_of[*deps.begin()];
    }
    CUstream st = streams[si];
    if (!forked[si]) {
      sfx::check_cu(d.cuStreamWaitEvent(st, ev_fork, 0), "cuStreamWaitEvent");
      forked[si] = true;
    }
    for (int q : deps)
      if (stream_of[q] != si) sfx::check_cu(d.cuStreamWaitEvent(st, G->branch_events[q], 0), "cuStreamWaitEvent");
    launch(k, gather_ptrs(G, k->src.inputs, where), gather_ptrs(G, k->src.outputs, where), st);
    sfx::check_cu(d.cuEventRecord(G->branch_events[p], st), "cuEventRecord");
    stream_of[p] = si;
  }
  for (size_t i = 1; i < streams.size(); ++i) {
    if (!forked[i]) continue;
    CUevent ev = G->branch_events[K + i];
    sfx::check_cu(d.cuEventRecord(ev, streams[i]), "cuEventRecord");
    sfx::check_cu(d.cuStreamWaitEvent(s, ev, 0), "cuStreamWaitEvent");
  }
}

}  // namespace

extern "C" {

int32_t sfx_abi_version(void) { return SFX_ABI_VERSION; }
const char* sfx_last_error(void) { return g_last_error.c_str(); }

sfx_status sfx_ctx_create(int32_t device, sfx_ctx** out) {
  return guard([&] {
    if (!out) throw sfx::Error(SFX_ERR_INVALID, "null out");
    const sfx::Driver& d = sfx::driver();
    auto c = std::make_unique<sfx_ctx>();
    c->device = device;
    sfx::check_cu(d.cuDeviceGet(&c->dev, device), "cuDeviceGet");
    sfx::check_cu(d.cuDevicePrimaryCtxRetain(&c->cu, c->dev), "cuDevicePrimaryCtxRetain");
    c->bind();
    *out = c.release();
  });
}

sfx_status sfx_ctx_destroy(sfx_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    try {
      ctx->bind();
      for (auto& [sz, p] : ctx->pool) sfx::driver().cuMemFree(p);
      for (auto& [p, sz] : ctx->live) sfx::driver().cuMemFree(p);
      for (CUdeviceptr p : ctx->peer_opened) sfx::driver().cuIpcCloseMemHandle(p);
      if (ctx->peer_table) sfx::driver().cuMemFree(ctx->peer_table);
      if (ctx->peer_base) sfx::driver().cuMemFree(ctx->peer_base);
    } catch (...) {
    }
    delete ctx;
  });
}

sfx_status sfx_alloc(sfx_ctx* ctx, uint64_t bytes, uint64_t* dptr) {
  return guard([&] {
    if (!ctx || !dptr) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    *dptr = ctx->alloc(bytes);
  });
}

sfx_status sfx_free(sfx_ctx* ctx, uint64_t dptr) {
  return guard([&] {
    if (!ctx) throw sfx::Error(SFX_ERR_INVALID, "null ctx");
    if (dptr) ctx->release(dptr);
  });
}

sfx_status sfx_host_alloc(sfx_ctx* ctx, uint64_t bytes, void** hptr) {
  return guard([&] {
    if (!ctx || !hptr) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    ctx->bind();
    sfx::check_cu(sfx::driver().cuMemHostAlloc(hptr, std::max<uint64_t>(bytes, 4), 0), "cuMemHostAlloc");
  });
}

sfx_status sfx_host_free(sfx_ctx* ctx, void* hptr) {
  return guard([&] {
    if (!ctx) throw sfx::Error(SFX_ERR_INVALID, "null ctx");
    ctx->bind();
    if (hptr) sfx::check_cu(sfx::driver().cuMemFreeHost(hptr), "cuMemFreeHost");
  });
}

sfx_status sfx_memcpy_h2d(sfx_ctx* ctx, uint64_t dst, const void* src, uint64_t bytes, void* stream) {
  return guard([&] {
    ctx->bind();
    sfx::check_cu(sfx::driver().cuMemcpyHtoDAsync(dst, src, bytes, static_cast<CUstream>(stream)), "cuMemcpyHtoDAsync");
  });
}

sfx_status sfx_memcpy_d2h(sfx_ctx* ctx, void* dst, uint64_t src, uint64_t bytes, void* stream) {
  return guard([&] {
    ctx->bind();
    sfx::check_cu(sfx::driver().cuMemcpyDtoHAsync(dst, src, bytes, static_cast<CUstream>(stream)), "cuMemcpyDtoHAsync");
  });
}

sfx_status sfx_memset_d32(sfx_ctx* ctx, uint64_t dst, uint32_t value, uint64_t count, void* stream) {
  return guard([&] {
    ctx->bind();
    sfx::check_cu(sfx::driver().cuMemsetD32Async(dst, value, count, static_cast<CUstream>(stream)), "cuMemsetD32Async");
  });
}

sfx_status sfx_stream_sync(sfx_ctx* ctx, void* stream) {
  return guard([&] {
    ctx->bind();
    sfx::check_cu(sfx::driver().cuStreamSynchronize(static_cast<CUstream>(stream)), "cuStreamSynchronize");
  });
}

int64_t sfx_launch_count(sfx_ctx* ctx) { return ctx ? ctx->launches.load() : -1; }

sfx_status sfx_program_compile(sfx_ctx* ctx, const sfx_graph_desc* graph, int32_t program_index,
                               const sfx_compile_opts* opts, sfx_kernel** out) {
  return guard([&] {
    if (!ctx || !out) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    sfx::Graph g = sfx::graph_from_desc(graph);
    *out = build_kernel(ctx, g, program_index, opts);
  });
}

sfx_status sfx_program_codegen(const sfx_graph_desc* graph, int32_t program_index, const sfx_compile_opts* opts,
                               char* source_out, uint64_t source_cap, char* cubin_path_out, uint64_t path_cap,
                               char* strategy_out, uint64_t strategy_cap) {
  return guard([&] {
    sfx::Graph g = sfx::graph_from_desc(graph);
    if (program_index >= static_cast<int32_t>(g.programs.size())) add_barrier_programs(g);
    sfx_compile_opts o{};
    if (opts) o = *opts;
    sfx::KernelSource ks = sfx::lower_program(g, program_index, o);
    sfx::Cubin cb = sfx::compile_cubin(ks.code, ks.entry, ks.nvrtc_options);
    auto put = [](char* dst, uint64_t cap, const std::string& s) {
      if (!dst || cap == 0) return;
      size_t n = std::min<size_t>(s.size(), cap - 1);
      std::memcpy(dst, s.data(), n);
      dst[n] = 0;
    };
    put(source_out, source_cap, ks.code);
    put(cubin_path_out, path_cap, cb.path);
    put(strategy_out, strategy_cap, ks.strategy + " " + ks.note);
  });
}

sfx_status sfx_program_signature(const sfx_graph_desc* graph, int32_t program_index, const sfx_compile_opts* opts,
                                 char* out, uint64_t cap) {
  return guard([&] {
    sfx::Graph g = sfx::graph_from_desc(graph);
    if (program_index >= static_cast<int32_t>(g.programs.size())) add_barrier_programs(g);
    sfx_compile_opts o{};
    if (opts) o = *opts;
    const std::string sig = sfx::kernel_signature(g, program_index, o);
    if (!out || cap <= sig.size()) throw sfx::Error(SFX_ERR_INVALID, "signature buffer too small");
    std::memcpy(out, sig.c_str(), sig.size() + 1);
  });
}

int32_t sfx_template_param_has(const char* signature) {
  return signature && sfx::template_param_find(signature) ? 1 : 0;
}

sfx_status sfx_template_param_put(const char* signature, int32_t rows_per_cta, int32_t threads_per_row,
                                  int32_t items_per_thread, int32_t pipe_ctas_per_sm, double tuned_us,
                                  double default_us, const char* source) {
  return guard([&] {
    if (!signature || !*signature) throw sfx::Error(SFX_ERR_INVALID, "empty signature");
    std::string src = source ? source : "";
    for (char& ch : src)
      if (ch == '|' || ch == '\n') ch = ' ';
    sfx::template_param_put(signature, rows_per_cta, threads_per_row, items_per_thread, pipe_ctas_per_sm, tuned_us,
                            default_us, src);
  });
}

sfx_status sfx_template_params_text(char* out, uint64_t cap, uint64_t* needed) {
  return guard([&] {
    const std::string t = sfx::template_params_text();
    if (needed) *needed = t.size() + 1;
    if (out && cap > t.size()) std::memcpy(out, t.c_str(), t.size() + 1);
  });
}

// Device timer for the perf-library miss path: one group compiled with `opts`,
// launched back to back on synthetic inputs (every element 0.5 / 1; rotating
// buffer sets when a set is smaller than 3x L2), CUDA events around `reps`
// launches.  *checksum = fp64 sum of output 0 of the first set (candidate
// kernels of one group must agree on it).
sfx_status sfx_program_time(sfx_ctx* ctx, const sfx_graph_desc* graph, int32_t program_index,
                            const sfx_compile_opts* opts, int32_t reps, double* us_out, double* checksum) {
  return guard([&] {
    if (!ctx || !us_out) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    sfx::Graph g = sfx::graph_from_desc(graph);
    if (program_index >= static_cast<int32_t>(g.programs.size())) add_barrier_programs(g);
    std::unique_ptr<sfx_kernel, void (*)(sfx_kernel*)> k(build_kernel(ctx, g, program_index, opts), destroy_kernel);
    const sfx::Driver& d = sfx::driver();
    ctx->bind();
    int l2 = 0;
    d.cuDeviceGetAttribute(&l2, CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE, ctx->dev);
    uint64_t per_set = 0;
    for (int n : k->src.inputs) per_set += g.nodes[n].numel() * 4;
    for (int n : k->src.outputs) per_set += g.nodes[n].numel() * 4;
    const int nsets = static_cast<int>(std::min<uint64_t>(8, std::max<uint64_t>(1, (3ull * l2 + per_set - 1) /
                                                                                      std::max<uint64_t>(per_set, 1))));
    std::vector<std::vector<CUdeviceptr>> ins(nsets), outs(nsets);
    CUstream s = nullptr;
    CUevent e0 = nullptr, e1 = nullptr;
    auto cleanup = [&] {
      for (auto& v : ins)
        for (CUdeviceptr p : v) ctx->release(p);
      for (auto& v : outs)
        for (CUdeviceptr p : v) ctx->release(p);
      if (e0) d.cuEventDestroy(e0);
      if (e1) d.cuEventDestroy(e1);
      if (s) d.cuStreamDestroy(s);
    };
    try {
      sfx::check_cu(d.cuStreamCreate(&s, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
      for (int i = 0; i < nsets; ++i) {
        for (int n : k->src.inputs) {
          CUdeviceptr p = ctx->alloc(g.nodes[n].numel() * 4);
          ins[i].push_back(p);
          const uint32_t bits = g.nodes[n].dtype == SFX_F32 ? 0x3f000000u : 1u;
          sfx::check_cu(d.cuMemsetD32Async(p, bits, g.nodes[n].numel(), s), "cuMemsetD32Async");
        }
        for (int n : k->src.outputs) outs[i].push_back(ctx->alloc(g.nodes[n].numel() * 4));
      }
      for (int i = 0; i < 3; ++i) launch(k.get(), ins[i % nsets], outs[i % nsets], s);
      sfx::check_cu(d.cuEventCreate(&e0, CU_EVENT_DEFAULT), "cuEventCreate");
      sfx::check_cu(d.cuEventCreate(&e1, CU_EVENT_DEFAULT), "cuEventCreate");
      const int r = std::max(1, reps);
      sfx::check_cu(d.cuEventRecord(e0, s), "cuEventRecord");
      for (int i = 0; i < r; ++i) launch(k.get(), ins[i % nsets], outs[i % nsets], s);
      sfx::check_cu(d.cuEventRecord(e1, s), "cuEventRecord");
      sfx::check_cu(d.cuEventSynchronize(e1), "cuEventSynchronize");
      float ms = 0;
      sfx::check_cu(d.cuEventElapsedTime(&ms, e0, e1), "cuEventElapsedTime");
      *us_out = 1000.0 * ms / r;
      if (checksum) {
        const int o = k->src.outputs.empty() ? -1 : k->src.outputs[0];
        double sum = 0;
        if (o >= 0) {
          const int64_t n = std::min<int64_t>(g.nodes[o].numel(), int64_t{16} << 20);
          std::vector<uint32_t> host(n);
          sfx::check_cu(d.cuMemcpyDtoH(host.data(), outs[(r - 1) % nsets][0], n * 4), "cuMemcpyDtoH");
          for (uint32_t bits : host) {
            if (g.nodes[o].dtype == SFX_F32) {
              float f;
              std::memcpy(&f, &bits, 4);
              sum += f;
            } else {
              sum += static_cast<int32_t>(bits);
            }
          }
        }
        *checksum = sum;
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

sfx_status sfx_kernel_get_info(sfx_kernel* k, sfx_kernel_info* info) {
  return guard([&] {
    if (!k || !info) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    info->strategy = k->src.strategy.c_str();
    info->entry = k->src.entry.c_str();
    info->n_inputs = static_cast<int32_t>(k->src.inputs.size());
    info->n_outputs = static_cast<int32_t>(k->src.outputs.size());
    info->grid = k->src.grid_x * k->src.grid_y;
    info->block = k->src.block;
    info->smem_bytes = k->src.smem;
    info->workspace_bytes = k->src.workspace_bytes;
    info->algorithmic_bytes = k->src.algorithmic_bytes;
    info->registers = k->regs;
    info->vector_width = k->src.vector_width;
  });
}

sfx_status sfx_kernel_input_instrs(sfx_kernel* k, int32_t* out, int32_t cap) {
  return guard([&] {
    if (!k || (!out && cap > 0)) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    for (size_t i = 0; i < k->src.inputs.size() && static_cast<int32_t>(i) < cap; ++i) out[i] = k->src.inputs[i];
  });
}

sfx_status sfx_program_launch(sfx_kernel* k, const uint64_t* inputs, int32_t n_inputs, const uint64_t* outputs,
                              int32_t n_outputs, void* stream) {
  return guard([&] {
    if (!k) throw sfx::Error(SFX_ERR_INVALID, "null kernel");
    k->ctx->bind();
    std::vector<CUdeviceptr> in(inputs, inputs + std::max(0, n_inputs));
    std::vector<CUdeviceptr> out(outputs, outputs + std::max(0, n_outputs));
    launch(k, in, out, static_cast<CUstream>(stream));
  });
}

sfx_status sfx_kernel_destroy(sfx_kernel* k) {
  return guard([&] { destroy_kernel(k); });
}

sfx_status sfx_graph_compile(sfx_ctx* ctx, const sfx_graph_desc* desc, const sfx_compile_opts* opts,
                             sfx_graph** out) {
  return guard([&] {
    if (!ctx || !out) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    auto G = std::make_unique<sfx_graph>();
    G->ctx = ctx;
    if (opts) G->opts = *opts;
    G->graph = sfx::graph_from_desc(desc);
    G->n_planned = static_cast<int>(G->graph.programs.size());
    add_barrier_programs(G->graph);
    for (size_t i = 0; i < G->graph.nodes.size(); ++i)
      if (G->graph.nodes[i].op == SFX_OP_PARAMETER) G->params.push_back(static_cast<int>(i));
    const sfx::Graph& g = G->graph;
    std::sort(G->params.begin(), G->params.end(), [&](int a, int b) { return g.nodes[a].id < g.nodes[b].id; });
    G->order = condensation_order(g);
    try {
      for (size_t p = 0; p < g.programs.size(); ++p)
        G->kernels.push_back(build_kernel(ctx, g, static_cast<int>(p), opts));
      // device-resident intermediates (roots consumed by later groups) and
      // dense constants; graph outputs and params come from the caller
      std::set<int> outs(g.outputs.begin(), g.outputs.end());
      const sfx::Driver& d = sfx::driver();
      for (const sfx::Program& p : g.programs)
        for (int r : p.roots)
          if (!outs.count(r)) G->mid_nodes.push_back(r);
      for (size_t i = 0; i < g.nodes.size(); ++i) {
        const sfx::Node& n = g.nodes[i];
        if (n.op != SFX_OP_CONSTANT || n.is_splat()) continue;
        bool used = outs.count(static_cast<int>(i)) > 0;
        for (const sfx::Program& p : g.programs)
          if (std::find(p.inputs.begin(), p.inputs.end(), static_cast<int>(i)) != p.inputs.end()) used = true;
        if (!used) continue;
        std::vector<uint32_t> host(n.numel());
        for (int64_t e = 0; e < n.numel(); ++e) {
          double raw = n.literal[e];
          if (n.dtype == SFX_F32) {
            float f = static_cast<float>(raw);
            std::memcpy(&host[e], &f, 4);
          } else {
            int32_t v = static_cast<int32_t>(raw);
            std::memcpy(&host[e], &v, 4);
          }
        }
        CUdeviceptr dp = ctx->alloc(n.numel() * 4);
        sfx::check_cu(d.cuMemcpyHtoDAsync(dp, host.data(), n.numel() * 4, nullptr), "cuMemcpyHtoDAsync");
        sfx::check_cu(d.cuStreamSynchronize(nullptr), "cuStreamSynchronize");
        G->owned[static_cast<int>(i)] = dp;
      }
      for (size_t i = 0; i < g.nodes.size(); ++i) {
        const sfx::Node& n = g.nodes[i];
        if (n.is_splat() && outs.count(static_cast<int>(i))) {
          CUdeviceptr dp = ctx->alloc(n.numel() * 4);
          float f = static_cast<float>(n.literal[0]);
          int32_t v = static_cast<int32_t>(n.literal[0]);
          uint32_t bits;
          if (n.dtype == SFX_F32) std::memcpy(&bits, &f, 4);
          else std::memcpy(&bits, &v, 4);
          sfx::check_cu(d.cuMemsetD32Async(dp, bits, n.numel(), nullptr), "cuMemsetD32Async");
          G->owned[static_cast<int>(i)] = dp;
        }
      }
    } catch (...) {
      for (sfx_kernel* k : G->kernels) destroy_kernel(k);
      for (auto& [n, p] : G->owned) ctx->release(p);
      throw;
    }
    *out = G.release();
  });
}

sfx_status sfx_graph_param_instrs(sfx_graph* G, int32_t* out, int32_t cap, int32_t* n) {
  return guard([&] {
    if (!G) throw sfx::Error(SFX_ERR_INVALID, "null graph");
    if (n) *n = static_cast<int32_t>(G->params.size());
    for (size_t i = 0; i < G->params.size() && static_cast<int32_t>(i) < cap; ++i) out[i] = G->params[i];
  });
}

sfx_status sfx_graph_kernel(sfx_graph* G, int32_t program_index, sfx_kernel** out) {
  return guard([&] {
    if (!G || !out) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    if (program_index < 0 || program_index >= static_cast<int32_t>(G->kernels.size()))
      throw sfx::Error(SFX_ERR_INVALID, "program index out of range");
    *out = G->kernels[program_index];
  });
}

sfx_status sfx_graph_kernel_count(sfx_graph* G, int32_t* n_kernels, int32_t* n_programs) {
  return guard([&] {
    if (!G) throw sfx::Error(SFX_ERR_INVALID, "null graph");
    if (n_kernels) *n_kernels = static_cast<int32_t>(G->kernels.size());
    if (n_programs) *n_programs = G->n_planned;
  });
}

sfx_status sfx_graph_run(sfx_graph* G, const uint64_t* params, int32_t n_params, const uint64_t* outputs,
                         int32_t n_outputs, void* stream, int32_t use_cuda_graph) {
  return guard([&] {
    if (!G) throw sfx::Error(SFX_ERR_INVALID, "null graph");
    if (n_params != static_cast<int32_t>(G->params.size()))
      throw sfx::Error(SFX_ERR_INVALID, "expected " + std::to_string(G->params.size()) + " params");
    if (n_outputs != static_cast<int32_t>(G->graph.outputs.size()))
      throw sfx::Error(SFX_ERR_INVALID, "expected " + std::to_string(G->graph.outputs.size()) + " outputs");
    std::lock_guard<std::mutex> lock(G->run_mu);
    G->ctx->bind();
    CUstream s = static_cast<CUstream>(stream);
    const sfx::Driver& d = sfx::driver();
    if (!use_cuda_graph) {
      graph_enqueue(G, params, outputs, s, mids_for(G, eager_key(s)));
      return;
    }
    if (!s) throw sfx::Error(SFX_ERR_INVALID, "CUDA-graph replay needs a non-default stream");
    std::vector<uint64_t> key(params, params + n_params);
    key.insert(key.end(), outputs, outputs + n_outputs);
    std::vector<uint64_t> mkey{1};
    mkey.insert(mkey.end(), key.begin(), key.end());
    const std::map<int, CUdeviceptr>& mid = mids_for(G, mkey);
    G->last_mid[s] = &mid;
    auto it = G->captured.find(key);
    if (it == G->captured.end()) {
      int64_t before = G->ctx->launches.load();
      // this capture's own workspaces, allocated and zeroed before capturing
      std::map<const sfx_kernel*, CUdeviceptr> cws;
      std::vector<CUdeviceptr>& owned_ws = G->captured_ws[key];
      for (sfx_kernel* k : G->kernels)
        if (k->src.workspace_bytes > 0 && k->src.peer_bytes == 0) {
          CUdeviceptr w = G->ctx->alloc(static_cast<uint64_t>(k->src.workspace_bytes));
          owned_ws.push_back(w);
          sfx::check_cu(d.cuMemsetD32Async(w, 0, (k->src.workspace_bytes + 3) / 4, s), "cuMemsetD32Async");
          cws[k] = w;
        }
      sfx::check_cu(d.cuStreamSynchronize(s), "cuStreamSynchronize");
      sfx::check_cu(d.cuStreamBeginCapture(s, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL), "cuStreamBeginCapture");
      CUgraph graph = nullptr;
      t_capture_ws = &cws;
      try {
        graph_enqueue(G, params, outputs, s, mid);
        t_capture_ws = nullptr;
      } catch (...) {
        t_capture_ws = nullptr;
        d.cuStreamEndCapture(s, &graph);
        if (graph) d.cuGraphDestroy(graph);
        for (CUdeviceptr w : owned_ws) G->ctx->release(w);
        G->captured_ws.erase(key);
        throw;
      }
      sfx::check_cu(d.cuStreamEndCapture(s, &graph), "cuStreamEndCapture");
      G->ctx->launches.store(before);  // captured, not launched
      CUgraphExec exec = nullptr;
      sfx::check_cu(d.cuGraphInstantiateWithFlags(&exec, graph, 0), "cuGraphInstantiate");
      it = G->captured.emplace(key, std::make_pair(graph, exec)).first;
    }
    sfx::check_cu(d.cuGraphLaunch(it->second.second, s), "cuGraphLaunch");
    G->ctx->launches.fetch_add(static_cast<int64_t>(G->order.size()));
  });
}

namespace {

// The host path (sfx_graph_run_host / _async): enqueues one run; on return
// every stream of the run is joined into `s` (the run is complete when `s` is).
void host_enqueue(sfx_graph* G, const void* const* params, int32_t n_params, void* const* outputs,
                  int32_t n_outputs, CUstream s) {
  if (!G) throw sfx::Error(SFX_ERR_INVALID, "null graph");
  if (n_params != static_cast<int32_t>(G->params.size()) ||
      n_outputs != static_cast<int32_t>(G->graph.outputs.size()))
    throw sfx::Error(SFX_ERR_INVALID, "param/output count mismatch");
  G->ctx->bind();
  const sfx::Driver& d = sfx::driver();
  const sfx::Graph& g = G->graph;
  const int K = static_cast<int>(G->kernels.size());
  sfx_graph::HostSlot& slot = G->hslot[G->hnext];
  G->hnext ^= 1;
  if (slot.bufs.empty()) {
    for (int p : G->params) slot.bufs.push_back(G->ctx->alloc(G->graph.nodes[p].numel() * 4));
    for (int o : G->graph.outputs) slot.bufs.push_back(G->ctx->alloc(G->graph.nodes[o].numel() * 4));
    slot.flags = G->ctx->alloc(static_cast<uint64_t>(K) * kFlagWords * 4);
    sfx::check_cu(d.cuEventCreate(&slot.free_ev, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  }
  std::vector<uint64_t> dp(slot.bufs.begin(), slot.bufs.begin() + n_params);
  std::vector<uint64_t> dout(slot.bufs.begin() + n_params, slot.bufs.end());
  if (!G->d2h) {
    sfx::check_cu(d.cuStreamCreate(&G->d2h, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    sfx::check_cu(d.cuStreamCreate(&G->h2d, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    sfx::check_cu(d.cuStreamCreate(&G->h2d2, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    sfx::check_cu(d.cuStreamCreate(&G->d2h2, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
    G->events.resize(3 * K + 2);
    for (CUevent& e : G->events) sfx::check_cu(d.cuEventCreate(&e, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    for (CUevent& e : G->join_ev) sfx::check_cu(d.cuEventCreate(&e, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    G->host_order = host_order(G);
    G->host_kernels.assign(K, nullptr);
    if (host_streaming() && !G->opts.debug_checks) {  // debug: every launch coverage-checked, whole copies
      sfx_compile_opts ho = G->opts;
      ho.host_stream = 1;
      for (int p = 0; p < K; ++p) {
        const std::string& st = G->kernels[p]->src.strategy;
        if (st != "row" && st != "map") continue;
        sfx_kernel* hk = build_kernel(G->ctx, g, p, &ho);
        if (hk->src.stream_R > 0) G->host_kernels[p] = hk;
        else destroy_kernel(hk);
      }
    }
  }
  // Overlapped host path.  Streams: host->device copies (h2d, h2d2), the
  // launches (s), device->host copies (d2h, d2h2).  A group whose template
  // works on an [R, C] row space (row / map, KernelSource::stream_R) is fed in
  // row chunks: a copy stream lands chunk j of its row-local inputs and sets
  // the group's gate[j] = 1 (cuStreamWriteValue32); the kernel's CTAs of chunk
  // j wait on gate[j], and each bumps done[j] once its rows are stored; a
  // copy-back stream waits for done[j] == the chunk's CTA count
  // (cuStreamWaitValue32) and returns chunk j of the group's graph outputs.
  // Chunks alternate between the two streams of each direction, so one
  // stream's copy runs while the other waits on its stream memory operation
  // (a memop drains the copy pipeline: ~20 us per chunk on one stream).
  // So a group's launch starts when its first chunk lands and its results
  // start crossing back while the rest of its inputs are still in flight —
  // still ONE launch per group.  Other groups: whole copies, ordered by events.
  // Groups that return the most bytes go first (any dependency-respecting
  // order gives the same values).
  // This slot's previous run (two runs ago) must be done with its buffers
  // and flags before anything of this run touches them; the flags are reset
  // on the first copy stream (not on `s`, whose previous run's kernels would
  // otherwise hold back this run's copies), and every stream of the run
  // starts behind the reset.
  if (slot.used) sfx::check_cu(d.cuStreamWaitEvent(G->h2d, slot.free_ev, 0), "cuStreamWaitEvent");
  slot.used = true;
  sfx::check_cu(d.cuMemsetD32Async(slot.flags, 0, static_cast<size_t>(K) * kFlagWords, G->h2d), "cuMemsetD32Async");
  CUevent ev_reset = G->events[3 * K];
  sfx::check_cu(d.cuEventRecord(ev_reset, G->h2d), "cuEventRecord");
  for (CUstream st : {s, G->h2d2, G->d2h, G->d2h2})
    sfx::check_cu(d.cuStreamWaitEvent(st, ev_reset, 0), "cuStreamWaitEvent");

  std::map<int, CUdeviceptr> where = G->owned;
  const std::map<int, CUdeviceptr>& mid = mids_for(G, eager_key(s));
  where.insert(mid.begin(), mid.end());
  G->last_mid[s] = &mid;
  std::map<int, int> param_slot, out_slot;
  for (int i = 0; i < n_params; ++i) where[G->params[i]] = dp[i], param_slot[G->params[i]] = i;
  for (int i = 0; i < n_outputs; ++i) where[g.outputs[i]] = dout[i], out_slot[g.outputs[i]] = i;
  std::vector<bool> copied(n_params, false), returned(n_outputs, false);
  // host->device copy of rows [r0, r1) of a node split into R rows (whole: 0, R, R)
  auto h2d_rows = [&](int node, int64_t R, int64_t r0, int64_t r1, CUstream st) {
    const int slot = param_slot.at(node);
    const uint64_t row = static_cast<uint64_t>(g.nodes[node].numel() / R) * 4;
    sfx::check_cu(d.cuMemcpyHtoDAsync(dp[slot] + r0 * row, static_cast<const char*>(params[slot]) + r0 * row,
                                      (r1 - r0) * row, st),
                  "cuMemcpyHtoDAsync");
  };
  auto d2h_rows = [&](int node, int64_t R, int64_t r0, int64_t r1, CUstream st) {
    const int slot = out_slot.at(node);
    const uint64_t row = static_cast<uint64_t>(g.nodes[node].numel() / R) * 4;
    sfx::check_cu(d.cuMemcpyDtoHAsync(static_cast<char*>(outputs[slot]) + r0 * row, dout[slot] + r0 * row,
                                      (r1 - r0) * row, st),
                  "cuMemcpyDtoHAsync");
  };
  auto is_host_param = [&](int n) {
    auto it = param_slot.find(n);
    return it != param_slot.end() && !copied[it->second];
  };
  for (size_t q = 0; q < G->host_order.size(); ++q) {
    const int pi = G->host_order[q];
    sfx_kernel* k = G->host_kernels[pi] ? G->host_kernels[pi] : G->kernels[pi];
    const sfx::KernelSource& ks = k->src;
    std::vector<int> ret;  // graph outputs this group returns
    for (int r : ks.outputs)
      if (out_slot.count(r) && !returned[out_slot[r]]) ret.push_back(r);
    std::set<int> chunked;
    for (int in : ks.stream_inputs)
      if (is_host_param(in)) chunked.insert(in);
    const int64_t R = ks.stream_R;
    bool streamed = R > 0 && host_streaming() && (!chunked.empty() || !ret.empty());
    for (int r : ret)
      if (streamed && g.nodes[r].numel() % R) streamed = false;
    // chunk rows: ~16 MB of streamed bytes per chunk, a multiple of the CTA
    // row unit, at most kFlagWords - 1 chunks
    int64_t rpc = R, nch = 1;
    if (streamed) {
      uint64_t bytes = 0;
      for (int in : chunked) bytes += g.nodes[in].numel() * 4;
      for (int r : ret) bytes += g.nodes[r].numel() * 4;
      // default: up to 32 chunks of >= 8 MB (measured: C1 67 MB flat at 4-8 MB
      // chunks, C4 / C4b 1.63 / 2.99 ms at 4 MB vs 1.58 / 2.87 at 8 MB, C2 537 MB
      // best at ~16 MB, C5's 3.2 GB probs_d flat from 16 to 100 MB)
      const uint64_t cb = host_chunk_bytes() ? host_chunk_bytes() : std::max<uint64_t>(8 << 20, bytes / 32);
      int64_t want = std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, static_cast<int64_t>(bytes / cb)));
      const int64_t unit = std::max<int64_t>(1, ks.stream_unit);
      rpc = ((R + want - 1) / want + unit - 1) / unit * unit;
      nch = (R + rpc - 1) / rpc;
      if (nch > kMaxChunks) streamed = false, rpc = R, nch = 1;
    }
    // inputs: everything not chunked goes first, whole
    for (int in : ks.inputs)
      if (is_host_param(in) && !(streamed && chunked.count(in))) {
        h2d_rows(in, 1, 0, 1, G->h2d);
        copied[param_slot[in]] = true;
      }
    StreamArgs sa;
    const CUdeviceptr gate = slot.flags + static_cast<uint64_t>(pi) * kFlagWords * 4;
    if (streamed) {
      // the whole inputs above precede every chunk gate on both streams
      sfx::check_cu(d.cuEventRecord(G->events[3 * q + 2], G->h2d), "cuEventRecord");
      sfx::check_cu(d.cuStreamWaitEvent(G->h2d2, G->events[3 * q + 2], 0), "cuStreamWaitEvent");
      for (int64_t j = 0; j < nch; ++j) {
        CUstream st = (j & 1) ? G->h2d2 : G->h2d;
        const int64_t r0 = j * rpc, r1 = std::min(R, r0 + rpc);
        for (int in : chunked) h2d_rows(in, R, r0, r1, st);
        sfx::check_cu(d.cuStreamWriteValue32(st, gate + 4 * j, 1u, CU_STREAM_WRITE_VALUE_DEFAULT),
                      "cuStreamWriteValue32");
      }
      for (int in : chunked) copied[param_slot[in]] = true;
      sa.gate = gate;
      sa.done = gate + 4 * kMaxChunks;
      sa.chunk_elems = static_cast<long long>(rpc * ks.stream_C);
    } else {
      // whole copies: on the first copy stream, plus anything the second
      // stream still has in flight for earlier groups
      sfx::check_cu(d.cuEventRecord(G->events[3 * q], G->h2d), "cuEventRecord");
      sfx::check_cu(d.cuStreamWaitEvent(s, G->events[3 * q], 0), "cuStreamWaitEvent");
      sfx::check_cu(d.cuEventRecord(G->events[3 * q + 2], G->h2d2), "cuEventRecord");
      sfx::check_cu(d.cuStreamWaitEvent(s, G->events[3 * q + 2], 0), "cuStreamWaitEvent");
    }
    launch(k, gather_ptrs(G, ks.inputs, where), gather_ptrs(G, ks.outputs, where), s, sa);
    if (ret.empty()) continue;
    if (streamed) {
      const int64_t E = ks.stream_cta_elems, C = ks.stream_C;
      for (int64_t j = 0; j < nch; ++j) {
        CUstream st = (j & 1) ? G->d2h2 : G->d2h;
        const int64_t r0 = j * rpc, r1 = std::min(R, r0 + rpc);
        const int64_t ctas = (r1 * C + E - 1) / E - (r0 * C) / E;
        sfx::check_cu(d.cuStreamWaitValue32(st, sa.done + 4 * j, static_cast<cuuint32_t>(ctas),
                                            CU_STREAM_WAIT_VALUE_GEQ),
                      "cuStreamWaitValue32");
        for (int r : ret) d2h_rows(r, R, r0, r1, st);
      }
    } else {
      sfx::check_cu(d.cuEventRecord(G->events[3 * q + 1], s), "cuEventRecord");
      sfx::check_cu(d.cuStreamWaitEvent(G->d2h, G->events[3 * q + 1], 0), "cuStreamWaitEvent");
      for (int r : ret) d2h_rows(r, 1, 0, 1, G->d2h);
    }
    for (int r : ret) returned[out_slot[r]] = true;
  }
  // graph outputs no group produces (a parameter or constant listed as output)
  bool tail = false;
  for (int i = 0; i < n_outputs; ++i) {
    if (returned[i]) continue;
    int o = g.outputs[i];
    if (is_host_param(o)) {
      h2d_rows(o, 1, 0, 1, G->h2d);
      copied[param_slot[o]] = true;
    }
    tail = true;
  }
  if (tail) {
    CUevent ev = G->events[3 * K + 1];
    sfx::check_cu(d.cuEventRecord(ev, G->h2d), "cuEventRecord");
    sfx::check_cu(d.cuStreamWaitEvent(s, ev, 0), "cuStreamWaitEvent");
    for (int i = 0; i < n_outputs; ++i) {
      if (returned[i]) continue;
      int o = g.outputs[i];
      CUdeviceptr src = param_slot.count(o) ? dp[param_slot[o]] : G->owned.count(o) ? G->owned.at(o) : 0;
      if (!src) throw sfx::Error(SFX_ERR_EXEC, "no value for graph output " + g.nodes[o].id);
      sfx::check_cu(d.cuMemcpyDtoHAsync(outputs[i], src, g.nodes[o].numel() * 4, s), "cuMemcpyDtoHAsync");
    }
  }
  // join: `s` waits for every copy stream; the slot is free once `s` is here
  for (int j = 0; j < 4; ++j) {
    CUstream st = j == 0 ? G->h2d : j == 1 ? G->h2d2 : j == 2 ? G->d2h : G->d2h2;
    sfx::check_cu(d.cuEventRecord(G->join_ev[j], st), "cuEventRecord");
    sfx::check_cu(d.cuStreamWaitEvent(s, G->join_ev[j], 0), "cuStreamWaitEvent");
  }
  sfx::check_cu(d.cuEventRecord(slot.free_ev, s), "cuEventRecord");
}

}  // namespace

sfx_status sfx_graph_run_host(sfx_graph* G, const void* const* params, int32_t n_params, void* const* outputs,
                              int32_t n_outputs, void* stream) {
  return guard([&] {
    if (!G) throw sfx::Error(SFX_ERR_INVALID, "null graph");
    std::lock_guard<std::mutex> lock(G->run_mu);
    CUstream s = static_cast<CUstream>(stream);
    host_enqueue(G, params, n_params, outputs, n_outputs, s);
    sfx::check_cu(sfx::driver().cuStreamSynchronize(s), "cuStreamSynchronize");
  });
}

sfx_status sfx_graph_run_host_async(sfx_graph* G, const void* const* params, int32_t n_params,
                                    void* const* outputs, int32_t n_outputs, void* stream) {
  return guard([&] {
    if (!G) throw sfx::Error(SFX_ERR_INVALID, "null graph");
    std::lock_guard<std::mutex> lock(G->run_mu);
    host_enqueue(G, params, n_params, outputs, n_outputs, static_cast<CUstream>(stream));
  });
}

sfx_status sfx_graph_fetch(sfx_graph* G, int32_t instr_index, void* host_out, uint64_t bytes, void* stream) {
  return guard([&] {
    if (!G || !host_out) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    const sfx::Graph& g = G->graph;
    if (instr_index < 0 || instr_index >= static_cast<int32_t>(g.nodes.size()))
      throw sfx::Error(SFX_ERR_INVALID, "instruction index out of range");
    const sfx::Node& n = g.nodes[instr_index];
    if (bytes != static_cast<uint64_t>(n.numel()) * 4)
      throw sfx::Error(SFX_ERR_INVALID, "fetch of " + n.id + ": expected " + std::to_string(n.numel() * 4) + " bytes");
    std::lock_guard<std::mutex> lock(G->run_mu);
    G->ctx->bind();
    CUstream s = static_cast<CUstream>(stream);
    CUdeviceptr src = 0;
    auto own = G->owned.find(instr_index);
    if (own != G->owned.end()) src = own->second;
    auto last = G->last_mid.find(s);
    if (!src && last != G->last_mid.end()) {
      auto it = last->second->find(instr_index);
      if (it != last->second->end()) src = it->second;
    }
    if (!src) {
      bool mid = std::find(G->mid_nodes.begin(), G->mid_nodes.end(), instr_index) != G->mid_nodes.end();
      throw sfx::Error(SFX_ERR_INVALID, mid ? "no run on this stream yet: " + n.id
                                            : n.id + " is not device-resident in the graph (a parameter, a graph "
                                                     "output or a folded splat: the caller holds it)");
    }
    const sfx::Driver& d = sfx::driver();
    sfx::check_cu(d.cuMemcpyDtoHAsync(host_out, src, bytes, s), "cuMemcpyDtoHAsync");
    sfx::check_cu(d.cuStreamSynchronize(s), "cuStreamSynchronize");
  });
}

sfx_status sfx_graph_destroy(sfx_graph* G) {
  return guard([&] {
    if (!G) return;
    try {
      G->ctx->bind();
      const sfx::Driver& d = sfx::driver();
      for (auto& [key, ge] : G->captured) {
        d.cuGraphExecDestroy(ge.second);
        d.cuGraphDestroy(ge.first);
      }
      for (CUevent e : G->events) d.cuEventDestroy(e);
      for (CUevent e : G->join_ev)
        if (e) d.cuEventDestroy(e);
      for (auto& sl : G->hslot)
        if (sl.free_ev) d.cuEventDestroy(sl.free_ev);
      if (G->d2h) d.cuStreamDestroy(G->d2h);
      for (CUstream st : {G->h2d, G->h2d2, G->d2h2})
        if (st) d.cuStreamDestroy(st);
      for (CUstream st : G->branch_streams) d.cuStreamDestroy(st);
      for (CUevent e : G->branch_events) d.cuEventDestroy(e);
    } catch (...) {
    }
    for (auto& sl : G->hslot) {
      if (sl.flags) G->ctx->release(sl.flags);
      for (CUdeviceptr p : sl.bufs) G->ctx->release(p);
    }
    for (auto& [key, ws] : G->captured_ws)
      for (CUdeviceptr w : ws) G->ctx->release(w);
    for (sfx_kernel* k : G->kernels) destroy_kernel(k);
    for (sfx_kernel* k : G->host_kernels) destroy_kernel(k);
    for (auto& [n, p] : G->owned) G->ctx->release(p);
    for (auto& [key, m] : G->mids)
      for (auto& [n, p] : m) G->ctx->release(p);
    delete G;
  });
}

sfx_status sfx_nccl_unique_id(void* id_out) {
  return guard([&] {
    nccl_id_t id;
    check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof id);
  });
}

sfx_status sfx_nccl_init(sfx_ctx* ctx, const void* id, int32_t nranks, int32_t rank) {
  return guard([&] {
    if (!ctx || !id) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    ctx->bind();
    nccl_id_t nid;
    std::memcpy(&nid, id, sizeof nid);
    check_nccl(nccl().CommInitRank(&ctx->comm, nranks, nid, rank), "ncclCommInitRank");
  });
}

sfx_status sfx_allreduce_sum_f32(sfx_ctx* ctx, uint64_t buf, uint64_t count, void* stream) {
  return guard([&] {
    if (!ctx || !ctx->comm) throw sfx::Error(SFX_ERR_NCCL, "NCCL communicator not initialised");
    ctx->bind();
    // ncclFloat32 = 7, ncclSum = 0
    check_nccl(nccl().AllReduce(reinterpret_cast<const void*>(buf), reinterpret_cast<void*>(buf), count, 7, 0,
                                ctx->comm, static_cast<CUstream>(stream)),
               "ncclAllReduce");
  });
}

sfx_status sfx_peer_create(sfx_ctx* ctx, uint64_t bytes, void* handle_out) {
  return guard([&] {
    if (!ctx || !handle_out) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    if (ctx->peer_base) throw sfx::Error(SFX_ERR_INVALID, "peer arena already created");
    static_assert(sizeof(CUipcMemHandle) == SFX_PEER_HANDLE_BYTES, "IPC handle size");
    ctx->bind();
    const sfx::Driver& d = sfx::driver();
    bytes = std::max<uint64_t>(4096, (bytes + 4095) / 4096 * 4096);
    // a dedicated allocation (not pooled): IPC exports whole allocations
    sfx::check_cu(d.cuMemAlloc(&ctx->peer_base, bytes), "cuMemAlloc(peer arena)");
    sfx::check_cu(d.cuMemsetD32Async(ctx->peer_base, 0, bytes / 4, nullptr), "cuMemsetD32Async");
    sfx::check_cu(d.cuStreamSynchronize(nullptr), "cuStreamSynchronize");
    CUipcMemHandle h;
    sfx::check_cu(d.cuIpcGetMemHandle(&h, ctx->peer_base), "cuIpcGetMemHandle");
    std::memcpy(handle_out, &h, sizeof(h));
    ctx->peer_bytes = bytes;
  });
}

sfx_status sfx_peer_open(sfx_ctx* ctx, const void* handles, int32_t nranks, int32_t rank) {
  return guard([&] {
    if (!ctx || !handles) throw sfx::Error(SFX_ERR_INVALID, "null argument");
    if (!ctx->peer_base) throw sfx::Error(SFX_ERR_INVALID, "sfx_peer_create first");
    if (ctx->peer_table) throw sfx::Error(SFX_ERR_INVALID, "peer group already open");
    if (nranks < 1 || nranks > SFX_PEER_MAX_RANKS || rank < 0 || rank >= nranks)
      throw sfx::Error(SFX_ERR_INVALID, "peer group of " + std::to_string(nranks) + " ranks (max " +
                                            std::to_string(SFX_PEER_MAX_RANKS) + "), rank " + std::to_string(rank));
    ctx->bind();
    const sfx::Driver& d = sfx::driver();
    std::vector<uint64_t> table(nranks);
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) {
        table[r] = ctx->peer_base;
        continue;
      }
      CUipcMemHandle h;
      std::memcpy(&h, static_cast<const char*>(handles) + static_cast<size_t>(r) * SFX_PEER_HANDLE_BYTES, sizeof(h));
      CUdeviceptr p = 0;
      sfx::check_cu(d.cuIpcOpenMemHandle(&p, h, CU_IPC_MEM_LAZY_ENABLE_PEER_ACCESS),
                    ("cuIpcOpenMemHandle(rank " + std::to_string(r) + ")").c_str());
      ctx->peer_opened.push_back(p);
      table[r] = p;
    }
    sfx::check_cu(d.cuMemAlloc(&ctx->peer_table, nranks * sizeof(uint64_t)), "cuMemAlloc(peer table)");
    sfx::check_cu(d.cuMemcpyHtoD(ctx->peer_table, table.data(), nranks * sizeof(uint64_t)), "cuMemcpyHtoD");
    ctx->pn = nranks;
    ctx->prank = rank;
  });
}

}  // extern "C"
