/* sfx.h — C ABI of the B200 stitched-group executor (libsfx.so).
 *
 * Drop-in boundary for the FusionStitching hot path.  The
 * reference planner stays on the reference side: compile_graph
 * (reference proj/src/pipeline.cpp:18-63) produces one KernelProgram per fused
 * group; this library replaces what runs it:
 *
 *   run_program(const KernelProgram&, const TensorGraph&, externals)
 *       reference proj/include/stitchfuse/exec.hpp:60-61, proj/src/exec.cpp:296-412
 *       -> sfx_program_compile + sfx_program_launch  (one sm_100a launch per group)
 *   run_compiled(const CompileReport&, const TensorGraph&, inputs)
 *       reference proj/include/stitchfuse/pipeline.hpp:50-51, proj/src/pipeline.cpp:65-133
 *       -> sfx_graph_compile + sfx_graph_run / sfx_graph_run_host
 *   TensorValue host vectors (exec.hpp:27-38)
 *       -> device buffers from sfx_alloc / sfx_memcpy_*; host arrays in sfx_graph_run_host
 *   ExecError (exec.hpp:21-23)
 *       -> nonzero sfx_status + sfx_last_error() (thread-local); no exceptions cross the ABI.
 *
 * The descriptors below are flat C mirrors of the reference types:
 *   sfx_instr    <- Instruction   (ir.hpp:82-99)
 *   sfx_stmt     <- Statement = MaterializeStmt | BarrierStmt | InlineBindingStmt
 *                   (kernelgen.hpp:25-45), with the member's Schedule (schedule.hpp:24-34)
 *   sfx_program  <- KernelProgram (kernelgen.hpp:48-54) + FusedComputation (fusion.hpp:20-25)
 *                   + SchedulePlan.blocks/block_threads (schedule.hpp:36-41)
 *   sfx_graph_desc <- TensorGraph (ir.hpp:103-125) + CompileReport.kernels (pipeline.hpp:33-40)
 * Instruction references are indices into sfx_graph_desc.instrs.  Ids are kept
 * only for error messages and for ordering: externals of a program are passed
 * in ascending id order (the std::map order of run_program's `externals`).
 * Splat constants are folded into the generated kernel and take no slot.
 *
 * Conventions: all calls are synchronous on the host except launches/copies,
 * which are enqueued on the given CUstream (a cudaStream_t may be passed);
 * 0 = default stream.  Device pointers are CUdeviceptr values carried as
 * uint64_t.  Every element is 4 bytes (f32 or i32), row-major, 16-byte-aligned
 * base pointers (sfx_alloc guarantees 256 B alignment).
 */
#ifndef SFX_H
#define SFX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define SFX_MAX_RANK 8
#define SFX_ABI_VERSION 3

typedef int32_t sfx_status; /* 0 = ok */
enum {
  SFX_OK = 0,
  SFX_ERR_INVALID = 1,     /* malformed descriptor / argument (ParseError-like) */
  SFX_ERR_UNSUPPORTED = 2, /* template forced where it does not apply; group shape outside the lowering */
  SFX_ERR_COMPILE = 3,     /* NVRTC / module load failure */
  SFX_ERR_CUDA = 4,        /* driver error */
  SFX_ERR_EXEC = 5,        /* ExecError analogue (missing external, ...) */
  SFX_ERR_NCCL = 6
};

/* Opcode (ir.hpp:41-52) */
enum {
  SFX_OP_PARAMETER = 0, SFX_OP_CONSTANT, SFX_OP_ELEMENTWISE, SFX_OP_RESHAPE, SFX_OP_BITCAST,
  SFX_OP_TRANSPOSE, SFX_OP_BROADCAST, SFX_OP_REDUCE, SFX_OP_BATCH_MATMUL, SFX_OP_LIBRARY_CALL
};
/* ElementwiseKind (ir.hpp:54-73) */
enum {
  SFX_EW_ADD = 0, SFX_EW_SUB, SFX_EW_MUL, SFX_EW_MAX, SFX_EW_MIN, SFX_EW_NEG, SFX_EW_COMPARE,
  SFX_EW_SELECT, SFX_EW_SCALE, SFX_EW_EXP, SFX_EW_LOG, SFX_EW_DIVIDE, SFX_EW_POWER, SFX_EW_TANH,
  SFX_EW_SQRT, SFX_EW_RSQRT
};
enum { SFX_REDUCE_SUM = 0, SFX_REDUCE_MAX, SFX_REDUCE_MIN }; /* Reducer (ir.hpp:75) */
/* LibraryCall callee (Instruction.callee, ir.hpp:97), carried in sfx_instr.kind:
 * "matmul" is executable (exec.cpp:207-209), "opaque" is a barrier only. */
enum { SFX_CALLEE_MATMUL = 0, SFX_CALLEE_OPAQUE = 1 };
enum { SFX_F32 = 0, SFX_I32 = 1 };                          /* ElementType (ir.hpp:19) */
enum { SFX_SCHED_ROW = 0, SFX_SCHED_COL = 1 };               /* SchedType (schedule.hpp:22) */
enum { SFX_STMT_MATERIALIZE = 0, SFX_STMT_BARRIER = 1, SFX_STMT_INLINE = 2 };
enum { SFX_DEST_SHARED = 0, SFX_DEST_OUTPUT = 1 };

typedef struct sfx_instr {
  const char* id;
  int32_t opcode;
  int32_t kind;     /* elementwise kind; SFX_CALLEE_* for library calls */
  int32_t dtype;
  int32_t rank;
  int64_t dims[SFX_MAX_RANK];
  int32_t n_operands;
  int32_t operands[3];
  int64_t permutation[SFX_MAX_RANK];        /* transpose */
  int32_t n_dim_map;
  int64_t broadcast_dim_map[SFX_MAX_RANK];  /* broadcast */
  int32_t n_reduce_dims;
  int64_t reduce_dims[SFX_MAX_RANK];        /* reduce */
  int32_t reducer;
  double scalar;                            /* scale */
  int64_t n_literal;                        /* constant: 1 = splat */
  const double* literal;
} sfx_instr;

typedef struct sfx_stmt {
  int32_t kind;       /* SFX_STMT_* */
  int32_t instr;      /* materialize / inline */
  int64_t split_dim;  /* materialize: Schedule */
  int64_t sword;
  int32_t sched_type;
  int32_t dest;       /* SFX_DEST_* */
  int64_t offset;     /* shared: arena byte offset */
  int64_t bytes;      /* shared: bytes per block */
  int32_t root_index; /* output */
} sfx_stmt;

/* The geometry the reference executor READS a materialised member with
 * (exec.cpp:320-324): KernelProgram.arena_offsets and
 * SchedulePlan.per_instruction.  Writes use the statement's own schedule and
 * destination; a program whose reads and writes disagree is what the
 * executor's stale-read / containment checks reject. */
typedef struct sfx_member_plan {
  int64_t arena_offset;  /* -1: not in the arena */
  int64_t split_dim;
  int64_t sword;
  int32_t sched_type;    /* SFX_SCHED_* */
} sfx_member_plan;

typedef struct sfx_program {
  int32_t n_members;
  const int32_t* members;     /* FusedComputation.members */
  int32_t n_roots;
  const int32_t* roots;       /* FusedComputation.roots (sorted ids) = output slot order */
  int32_t fusion_root;
  int64_t blocks;             /* SchedulePlan.blocks */
  int32_t block_threads;      /* SchedulePlan.block_threads */
  int64_t arena_bytes;        /* KernelProgram.arena_bytes */
  int32_t n_stmts;
  const sfx_stmt* stmts;      /* KernelProgram.statements */
  const sfx_member_plan* member_plans; /* per member (members[] order); NULL = the statements' geometry */
} sfx_program;

typedef struct sfx_graph_desc {
  int32_t n_instrs;
  const sfx_instr* instrs;    /* TensorGraph.instructions() */
  int32_t n_outputs;
  const int32_t* outputs;     /* TensorGraph.outputs() */
  int32_t n_programs;
  const sfx_program* programs;/* CompileReport.kernels[i].program */
} sfx_graph_desc;

/* Lowering options. */
enum {
  SFX_STRATEGY_AUTO = 0,    /* pick map/row/col/colbc template (or dot for fuse_dot groups), else literal */
  SFX_STRATEGY_LITERAL = 1, /* literal KernelProgram lowering (reference chunking and fold order) */
  SFX_STRATEGY_MAP = 2,
  SFX_STRATEGY_ROW = 3,
  SFX_STRATEGY_COL = 4,
  SFX_STRATEGY_COLBC = 5    /* column reductions broadcast back (batch-norm): grid barriers, one launch; also the
                               split layout [A | K | B] (batch-norm over NCHW): a cluster or CTA per channel */
};
typedef struct sfx_compile_opts {
  int32_t strategy;      /* SFX_STRATEGY_* ; forcing an inapplicable one fails with SFX_ERR_UNSUPPORTED */
  int32_t debug_checks;  /* 1 = coverage check after every launch (the device twin of the reference's
                            coverage bitmap, exec.cpp:393-410): outputs are pre-filled with a canary,
                            and any element the kernel left unwritten (canary still there after two
                            launches with different canaries) fails the launch with SFX_ERR_EXEC
                            "incomplete coverage"; synchronous, not inside CUDA-graph capture.
                            2 = same, but the launch drops its last CTA (test hook: must be caught) */
  int32_t rows_per_cta;  /* 0 = auto (row template) */
  int32_t threads_per_row; /* 0 = auto (row template) */
  int32_t items_per_thread; /* 0 = auto (map template: 128-bit vectors per thread) */
  int32_t row_pipeline;     /* row template: 0 = auto, 1 = register-resident rows, 2 = TMA-staged pipeline, 4 = resident rows (all of a CTA's rows staged at entry) where applicable */
  int32_t pipe_warps;       /* TMA row pipeline: warps per CTA (0 = auto) */
  int32_t pipe_stages;      /* TMA row pipeline: row buffers per warp (0 = auto) */
  int32_t pipe_ctas_per_sm; /* TMA row pipeline: persistent CTAs per SM (0 = auto) */
  int32_t cross_rank;       /* 1 = this graph is one rank's batch shard: reductions over dim 0 combine
                               across the context's peer group inside the column kernel (peer memory,
                               see sfx_peer_*); other reductions over dim 0 are SFX_ERR_UNSUPPORTED */
  int32_t host_stream;      /* 1 = row / map kernels carry the host-streaming gate and completion code
                               (sfx_graph_run_host compiles these variants itself on first use; the
                               device-path kernels stay free of it) */
} sfx_compile_opts;

typedef struct sfx_ctx sfx_ctx;
typedef struct sfx_kernel sfx_kernel;
typedef struct sfx_graph sfx_graph;

/* Kernel facts for logging / measurement. */
typedef struct sfx_kernel_info {
  const char* strategy;      /* "map" | "row" | "col" | "colbc" | "literal" | "dot" */
  const char* entry;         /* kernel symbol */
  int32_t n_inputs;
  int32_t n_outputs;
  int64_t grid;              /* CTAs */
  int32_t block;             /* threads per CTA */
  int32_t smem_bytes;        /* dynamic shared memory */
  int64_t workspace_bytes;   /* device scratch owned by the kernel (cross-CTA partials) */
  int64_t algorithmic_bytes; /* non-splat external inputs read once + roots written once */
  int32_t registers;         /* per thread, from the loaded module */
  int32_t vector_width;      /* elements per 128-bit access on the main stream (1 or 4) */
} sfx_kernel_info;

/* ---- context / memory (device buffer manager) ---- */
int32_t sfx_abi_version(void);
const char* sfx_last_error(void);
sfx_status sfx_ctx_create(int32_t device, sfx_ctx** out);
sfx_status sfx_ctx_destroy(sfx_ctx* ctx);
sfx_status sfx_alloc(sfx_ctx* ctx, uint64_t bytes, uint64_t* dptr);
sfx_status sfx_free(sfx_ctx* ctx, uint64_t dptr);
sfx_status sfx_host_alloc(sfx_ctx* ctx, uint64_t bytes, void** hptr); /* pinned */
sfx_status sfx_host_free(sfx_ctx* ctx, void* hptr);
sfx_status sfx_memcpy_h2d(sfx_ctx* ctx, uint64_t dst, const void* src, uint64_t bytes, void* stream);
sfx_status sfx_memcpy_d2h(sfx_ctx* ctx, void* dst, uint64_t src, uint64_t bytes, void* stream);
sfx_status sfx_memset_d32(sfx_ctx* ctx, uint64_t dst, uint32_t value, uint64_t count, void* stream);
sfx_status sfx_stream_sync(sfx_ctx* ctx, void* stream);
/* Counters of kernels this library launched (monotonic, per context). */
int64_t sfx_launch_count(sfx_ctx* ctx);

/* ---- one fused group: replaces run_program (exec.cpp:296-412) ---- */
/* Lower program `program_index` of `graph` to CUDA, JIT it for sm_100a and load it. */
sfx_status sfx_program_compile(sfx_ctx* ctx, const sfx_graph_desc* graph, int32_t program_index,
                               const sfx_compile_opts* opts, sfx_kernel** out);
/* Lower + compile to a cubin only (no device needed); writes the CUDA source to
 * `source_out` (may be NULL) and the cubin path to `cubin_path_out` (may be NULL).
 * program_index >= n_programs selects the unfused instructions, as in sfx_graph_kernel. */
sfx_status sfx_program_codegen(const sfx_graph_desc* graph, int32_t program_index,
                               const sfx_compile_opts* opts, char* source_out, uint64_t source_cap,
                               char* cubin_path_out, uint64_t path_cap, char* strategy_out,
                               uint64_t strategy_cap);
sfx_status sfx_kernel_get_info(sfx_kernel* k, sfx_kernel_info* info);

/* ---- measured perf library (the paper's library-miss path: build, run and
 * time a kernel, record it; reference tuning.cpp:192-201 fills misses with an
 * analytical estimate instead) ---- */
/* Device timer: compiles program `program_index` with `opts`, launches it
 * `reps` times back to back on synthetic inputs and returns the average
 * per-launch time in microseconds; *checksum (may be NULL) = fp64 sum of
 * output 0, for checking that candidate lowerings agree. */
sfx_status sfx_program_time(sfx_ctx* ctx, const sfx_graph_desc* graph, int32_t program_index,
                            const sfx_compile_opts* opts, int32_t reps, double* us_out, double* checksum);
/* Template parameter cache (the B200 side of the perf library): groups are
 * filed under the signature of the kernel their default options generate;
 * lowering with default options uses a group's recorded parameters. */
sfx_status sfx_program_signature(const sfx_graph_desc* graph, int32_t program_index, const sfx_compile_opts* opts,
                                 char* out, uint64_t cap);
int32_t sfx_template_param_has(const char* signature);
sfx_status sfx_template_param_put(const char* signature, int32_t rows_per_cta, int32_t threads_per_row,
                                  int32_t items_per_thread, int32_t pipe_ctas_per_sm, double tuned_us,
                                  double default_us, const char* source);
/* The whole cache in its file format (SFX_TEMPLATE_PARAMS / template_params.txt);
 * *needed = bytes including the terminator. */
sfx_status sfx_template_params_text(char* out, uint64_t cap, uint64_t* needed);
/* Instruction indices of the input slots (ascending external id, splats excluded). */
sfx_status sfx_kernel_input_instrs(sfx_kernel* k, int32_t* out, int32_t cap);
/* One launch.  inputs: device pointers per input slot; outputs: per root (comp.roots order). */
sfx_status sfx_program_launch(sfx_kernel* k, const uint64_t* inputs, int32_t n_inputs,
                              const uint64_t* outputs, int32_t n_outputs, void* stream);
sfx_status sfx_kernel_destroy(sfx_kernel* k);

/* ---- whole compiled module: replaces run_compiled (pipeline.cpp:65-133) ---- */
sfx_status sfx_graph_compile(sfx_ctx* ctx, const sfx_graph_desc* graph, const sfx_compile_opts* opts,
                             sfx_graph** out);
/* Parameter slots: graph Parameters in ascending id order.  Output slots: graph.outputs order. */
sfx_status sfx_graph_param_instrs(sfx_graph* g, int32_t* out, int32_t cap, int32_t* n);
sfx_status sfx_graph_kernel(sfx_graph* g, int32_t program_index, sfx_kernel** out);
/* Kernels per run: n_programs planned groups + unfused instructions (see sfx_graph_run). */
sfx_status sfx_graph_kernel_count(sfx_graph* g, int32_t* n_kernels, int32_t* n_programs);
/* Device-resident run: params and outputs are device pointers; intermediates
 * between groups stay in HBM (pooled).  Launches one kernel per group in the
 * reference's condensation (Kahn) order, plus one per instruction the planner
 * left unfused (matmul barriers — BatchMatMul with fuse_dot off, LibraryCall
 * "matmul" — and stray shape ops; the reference runs them through eval_dense,
 * pipeline.cpp:124-127); those are the kernels program_index >= n_programs of
 * sfx_graph_kernel.  use_cuda_graph=1 replays
 * a captured CUDA graph for this exact pointer set (captured on first use). */
/* Concurrency: kernels that own a workspace (column / colbc cross-CTA
 * combine) get one workspace per stream, and a graph's intermediates (group
 * roots consumed by later groups) are one set per stream, so launches of one
 * kernel or graph on different streams may run concurrently (each with its own
 * buffers).  Every CUDA graph captured by sfx_graph_run owns its workspaces and
 * intermediates (replays of one capture are serialised by CUDA).  Exceptions: cross_rank kernels use one
 * workspace and one peer region and must run in the same order on every rank,
 * never concurrently with themselves; a launch captured by the CALLER's own
 * stream capture uses the kernel's default workspace, so such captured
 * replays must not overlap other launches of that kernel.  Calls on one
 * sfx_graph from several host threads are serialised internally. */
sfx_status sfx_graph_run(sfx_graph* g, const uint64_t* params, int32_t n_params,
                         const uint64_t* outputs, int32_t n_outputs, void* stream,
                         int32_t use_cuda_graph);
/* Host-buffer run (the TensorValue-in/TensorValue-out call): copies params
 * host->device, runs, copies outputs device->host, synchronizes the stream. */
sfx_status sfx_graph_run_host(sfx_graph* g, const void* const* params, int32_t n_params,
                              void* const* outputs, int32_t n_outputs, void* stream);
/* The same run, enqueued without waiting: complete when `stream` is (every
 * copy stream of the run is joined into it).  The graph stages host runs in
 * two device slots used alternately, so consecutive async runs overlap (run
 * i+1's host->device copies under run i's kernels and device->host copies).
 * Host buffers must be pinned (sfx_host_alloc or cudaHostRegister'ed) and stay
 * valid until the stream reaches the run. */
sfx_status sfx_graph_run_host_async(sfx_graph* g, const void* const* params, int32_t n_params,
                                    void* const* outputs, int32_t n_outputs, void* stream);
/* Read back a value the latest run on `stream` left in HBM: a group root that
 * is not a graph output (an intermediate between groups) or a dense constant.
 * This is how the binding returns run_compiled's full value map
 * (pipeline.cpp:104-118: every parameter, constant, singleton and group root)
 * without downloading intermediates on every run.  Synchronous.  Parameters,
 * graph outputs and splat constants are rejected: the caller holds them. */
sfx_status sfx_graph_fetch(sfx_graph* g, int32_t instr_index, void* host_out, uint64_t bytes, void* stream);
sfx_status sfx_graph_destroy(sfx_graph* g);

/* ---- collectives (batch-crossing column reduce) ---- */
#define SFX_NCCL_ID_BYTES 128
sfx_status sfx_nccl_unique_id(void* id_out /* SFX_NCCL_ID_BYTES */);
sfx_status sfx_nccl_init(sfx_ctx* ctx, const void* id, int32_t nranks, int32_t rank);
sfx_status sfx_allreduce_sum_f32(sfx_ctx* ctx, uint64_t buf, uint64_t count, void* stream);

/* Peer-memory group: the fused alternative to compute-then-allreduce.  Every
 * rank allocates a symmetric peer arena (same size on every rank), exchanges
 * the IPC handles out of band (torch.distributed / MPI / files) and opens the
 * others'.  Column kernels compiled afterwards with cross_rank=1 then push
 * their per-column partials into every rank's arena over NVLink (plain
 * stores + a release flag per column tile) and fold the ranks in rank order
 * inside the same launch, so all ranks get bit-identical results with no
 * separate collective.  Arena regions are assigned in kernel build order, so
 * every rank must compile the same graphs in the same order.  Replaces the
 * ncclAllReduce that would follow the reference's column reduce
 * (SURVEY §8(e)); the reference itself is single-process. */
#define SFX_PEER_HANDLE_BYTES 64
#define SFX_PEER_MAX_RANKS 8
sfx_status sfx_peer_create(sfx_ctx* ctx, uint64_t bytes, void* handle_out /* SFX_PEER_HANDLE_BYTES */);
sfx_status sfx_peer_open(sfx_ctx* ctx, const void* handles /* nranks x SFX_PEER_HANDLE_BYTES, rank order */,
                         int32_t nranks, int32_t rank);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* SFX_H */
