// Reference-side binding for the B200 executor: the code a maintainer of the
// reference adds so that existing callers of stitchfuse::run_program /
// stitchfuse::run_compiled run every fusion group as one sm_100a kernel.
//
// It is compiled against the reference headers (proj/include/stitchfuse) and
// links libsfx.so through the C ABI in include/sfx.h; see INTEGRATION.md.
// Signatures are those of reference exec.hpp:60-61 and pipeline.hpp:50-51.
#pragma once

#include <map>
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
// Returns the graph outputs (the values callers of the reference read).
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

}  // namespace stitchfuse_device
