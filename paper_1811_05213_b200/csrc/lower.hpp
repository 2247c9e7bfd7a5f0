// Fusion-group -> sm_100a kernel lowering (the subsystem BASELINE.json's
// north_star says changes: schedule selection per group, launch dimensions,
// shared-memory allocation across the stitched ops).  Input is one reference
// KernelProgram (reference proj/include/stitchfuse/kernelgen.hpp:48-54); output
// is the CUDA source of ONE stitched kernel plus its launch geometry.
//
// Strategies (chosen by GroupAnalyzer = analyze_* below):
//   map     — no reductions: 1-D kLoop over root elements, 128-bit vector
//             loads/stores, everything thread-composed in registers.
//   row     — reductions over trailing dims (LayerNorm, softmax): a thread
//             group per row, row held in registers, warp-shuffle combine,
//             reduced scalars broadcast back through registers.
//   col     — reductions over leading dims (bias-grad): column tiles x row
//             stripes, shared-memory partials, single-launch deterministic
//             cross-CTA combine (last-CTA ticket), elementwise roots written in
//             the same pass.
//   dot     — a lone matmul: an unfused barrier (BatchMatMul with fuse_dot
//             off, LibraryCall "matmul") that the reference runs through
//             eval_dense, or a fuse_dot group with nothing else in it:
//             register-tiled SIMT kernel, bit-exact k order (dot.cpp).
//             Groups that stitch other members to a BatchMatMul run on the
//             literal tier.
//   literal — any plan the reference emits: the KernelProgram executed as
//             written (reference blocks/chunk_box/arena/barriers, reference
//             fold order) with the arena in shared memory.  Correctness tier.
#pragma once

#include <string>
#include <vector>

#include "ir.hpp"

namespace sfx {

struct KernelSource {
  std::string strategy;
  std::string entry;
  std::string code;          // complete CUDA translation unit (prelude included)
  int64_t grid_x = 1, grid_y = 1;
  int block = 256;
  int smem = 0;              // dynamic shared memory bytes
  int64_t workspace_bytes = 0;
  bool cooperative = false;  // grid-wide barriers: launched cooperatively (co-residency checked)
  int cluster = 1;           // thread-block cluster size (__cluster_dims__); > 8 needs the non-portable opt-in
  // cross-rank column combine (opts.cross_rank): bytes of the symmetric peer
  // arena this kernel needs; the kernel then takes (peers, peer_off, rank,
  // nranks) after ws
  int64_t peer_bytes = 0;
  // host streaming (sfx_graph_run_host): the group's work is an [R, C] row
  // space (stream_R > 0) that the kernel can consume in row chunks as the
  // host->device copies land.  The kernel then takes (sgate, sdone, schunk)
  // after ws / the peer params: a CTA waits until *sgate > its chunk (the copy
  // stream bumps it after each chunk of `stream_inputs`), and bumps
  // sdone[chunk] when its rows are stored (the copy-back stream waits on it).
  // A CTA covers stream_cta_elems consecutive elements of the row space, so
  // chunks of a multiple of stream_unit rows never share a CTA.
  int64_t stream_R = 0, stream_C = 0, stream_cta_elems = 0, stream_unit = 0;
  std::vector<int> stream_inputs;  // row-local inputs: chunk j = rows [j*rpc, (j+1)*rpc)
  std::vector<int> inputs;   // node ids per input slot (Program::inputs)
  std::vector<int> outputs;  // node ids per output slot (Program::roots)
  int64_t algorithmic_bytes = 0;
  int vector_width = 1;
  std::string note;          // why this strategy / geometry
  // extra NVRTC options; see the i32 min/max note in lower.cpp
  std::vector<std::string> nvrtc_options;
};

KernelSource lower_program(const Graph& g, int program_index, const sfx_compile_opts& opts);

// Template parameter cache (lower.cpp): the signature a group's default-option
// kernel is filed under, lookups, in-process inserts and the text form.
std::string kernel_signature(const Graph& g, int program_index, const sfx_compile_opts& opts);
bool template_param_find(const std::string& sig);
void template_param_put(const std::string& sig, int rows_per_cta, int threads_per_row, int items_per_thread,
                        int pipe_ctas_per_sm, double tuned_us, double default_us, const std::string& source);
std::string template_params_text();

// Strategy the analyzer would pick (without generating code), with the reason
// the faster templates were rejected.
std::string choose_strategy(const Graph& g, int program_index, std::string* why);

// The matmul barrier kernel (dot.cpp).
KernelSource lower_dot(const Graph& g, const Program& p);
// fuse_dot group: a matmul (only root) whose operands are stitched elementwise / layout
// members, computed where the operand tiles are staged
bool dot_prologue_ok(const Graph& g, const Program& p, std::string* why);
KernelSource lower_dot_prologue(const Graph& g, const Program& p);

// A program whose only member is a matmul: an unfused barrier, or a fuse_dot
// group with nothing stitched to the BatchMatMul.  Runs the dot kernel.
bool dot_alone(const Graph& g, const Program& p);
bool is_matmul(const Node& n);

// Synthetic one-member program for an instruction the planner left unfused
// (Program::barrier set; includes a literal-tier plan).
Program barrier_program(const Graph& g, int node);

extern const char* kPrelude;

}  // namespace sfx
