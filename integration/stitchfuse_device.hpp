// Reference-side binding for the B200 executor: the code a maintainer of the
// reference adds so that existing callers of stitchfuse::run_program /
// stitchfuse::run_compiled run every fusion group as one sm_100a kernel.
//
// It is compiled against the reference headers (proj/include/stitchfuse) and
// links libsfx.so through the C ABI in include/sfx.h; see INTEGRATION.md.
// Signatures are those of reference exec.hpp:60-61 and pipeline.hpp:50-51.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "stitchfuse/exec.hpp"
#include "stitchfuse/pipeline.hpp"

namespace stitchfuse_device {

using stitchfuse::CompileReport;
using stitchfuse::InstrId;
using stitchfuse::KernelProgram;
using stitchfuse::TensorGraph;
using stitchfuse::TensorValue;

// Device twin of stitchfuse::run_program (exec.hpp:60-61): one stitched launch;
// returns one value per root in comp.roots order.  Throws stitchfuse::ExecError.
std::vector<TensorValue> run_program(const KernelProgram& program, const TensorGraph& graph,
                                     const std::map<InstrId, TensorValue>& externals);

// Device twin of stitchfuse::run_compiled (pipeline.hpp:50-51): one launch per
// CompiledKernel in condensation order, intermediates resident in HBM.
// Returns the reference's whole map (pipeline.cpp:104-118): every parameter,
// constant, unfused instruction and group root; the graph outputs come back
// with the run, other roots are read back from HBM afterwards.
std::map<InstrId, TensorValue> run_compiled(const CompileReport& report, const TensorGraph& graph,
                                            const std::map<InstrId, TensorValue>& inputs);

// Number of kernels the device executor launched so far (plan-parity check).
long long launches();

// Number of plans compiled so far.  Compiled kernels / modules are cached by
// plan signature (graph + program + options), so repeated run_program /
// run_compiled calls on the same plan reuse them: no re-lowering, no NVRTC,
// no module load, no device allocation.
long long compiles();

// Lowering tier for subsequent calls (SFX_STRATEGY_AUTO by default).
void set_strategy(int sfx_strategy);

// sfx_compile_opts.debug_checks for subsequent calls: 1 = the coverage check of
// the reference executor (exec.cpp:393-410) around every launch.
void set_debug_checks(int level);

// ---- measured perf library: the paper's library-miss path on the B200 ----
// (on a miss, build, run and time the kernel, record it.
// The reference's lookup_or_estimate, tuning.cpp:192-201, records an
// analytical estimate marked synthetic instead.)
struct MeasureStats {
  int keys_missed = 0;    // perf keys the planner looked up without a measured entry
  int keys_measured = 0;  // of those, timed on the device and recorded (synthetic = false)
  int groups_tuned = 0;   // planned groups whose template parameters were measured on miss
  int groups_changed = 0; // ... where a candidate beat the default parameters (>= 2%)
  std::vector<std::string> notes;
};

// Plans `graph` with `lib`; every key the planner missed (lookup_or_estimate
// inserted a synthetic estimate for it) is measured: the instruction alone,
// run under exactly that key's schedule and block size by the literal tier
// (the reference's chunk_box blocks, so the cost is schedule-sensitive), and
// recorded in `lib` in the reference's own format.  Re-planning with `lib`
// then hits on every key.  `max_keys` < 0: no limit.
MeasureStats measure_misses(const TensorGraph& graph, const stitchfuse::PipelineOptions& options,
                            stitchfuse::PerfLibrary& lib, const stitchfuse::CostModelParams& params, int reps = 10,
                            int max_keys = -1);

// Template parameters of the report's planned groups, measured on miss in the
// B200 template parameter cache: a group not in the cache (keyed by its
// default kernel's signature) is timed with its default parameters and every
// candidate of its template; the winner (>= 2% faster with the same output
// checksum, else the defaults) is recorded, so later lowerings of that group
// use it.  Returns what was tuned.
MeasureStats tune_templates(const CompileReport& report, const TensorGraph& graph, int reps = 20);

// The template parameter cache in its file format (write it where
// SFX_TEMPLATE_PARAMS points to persist it).
std::string template_params_text();

}  // namespace stitchfuse_device
