// TEST INFRASTRUCTURE — the reference's own executor tests, replayed through
// the device executor via the reference-side binding (integration/).
// Everything here is reference code or reference types: random graphs from
// tests/support.cpp:168-284, inputs from random_inputs (:286-298), plans from
// compile_graph / resolve_schedule / plan_shared_memory / emit_program, the
// oracle is the reference's interpret, the check is the reference's
// values_close(…, 1e-5) (:300-316).
//
//   device_parity random <seed> <count> [--fuse-dot-alternate] [--literal]
//        test_pipeline.cpp:106-123 / test_acceptance.cpp:41-62 (criterion 2)
//   device_parity schedules [--literal]
//        test_exec.cpp:108-137: every satisfiable root schedule of the
//        device-eligible fixtures runs and equals interpret
//   device_parity shrink [--literal]
//        test_exec.cpp:139-155: lowered smem limits (shrunk plans) keep outputs
//   device_parity crit9 | crit7
//        acceptance criteria 9 (50 fuse_dot executor runs, coverage-checked)
//        and 7 (shrunk fuse_dot fixture), test_acceptance.cpp:276-391
//   device_parity perflib <graph.json> <lib_out> <template_params_out> [max_keys]
//        the measured perf library: misses measured on the device, re-plan hits
//   device_parity cache
//        the binding's compiled-plan cache: one compile per plan signature
//   device_parity selfchecks
//        test_exec.cpp:157-194: the reference's corrupted programs throw
//        ExecError from both executors, with the same message
// Prints one JSON line; exit 0 iff every eligible case passed.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <set>
#include <sstream>

#include "../../integration/stitchfuse_device.hpp"
#include "json.hpp"
#include "sfx.h"
#include "stitchfuse/fixtures.hpp"
#include "stitchfuse/pipeline.hpp"
#include "support.hpp"

extern "C" {
#include "../sfx_oracle.h"
}

using namespace stitchfuse;
using json = nlohmann::json;

namespace {

// Everything the reference can execute: only "opaque" library calls are not
// (exec.cpp:207-209).
bool eligible(const TensorGraph& g) {
  for (const Instruction& i : g.instructions())
    if (i.opcode == Opcode::LibraryCall && i.callee != "matmul") return false;
  return true;
}

// Launches per run_compiled: one per planned group plus one per unfused
// instruction (matmul barriers and stray shape ops, which the reference
// evaluates densely, pipeline.cpp:124-127).
long long expected_launches(const CompileReport& report) {
  return static_cast<long long>(report.kernels.size() + report.fusion.unfused.size());
}

struct Tally {
  int cases = 0, passed = 0;
  json failures = json::array();
  void fail(const std::string& what) {
    if (failures.size() < 20) failures.push_back(what);
  }
};

// fp64 restatement of the graph (oracle/sfx_oracle.c, mode 1) for the
// reduction-order tolerance policy.
std::map<InstrId, TensorValue> interpret_fp64(const TensorGraph& g, const std::map<InstrId, TensorValue>& inputs) {
  const auto& ins = g.instructions();
  std::map<InstrId, int32_t> index;
  for (size_t i = 0; i < ins.size(); ++i) index[ins[i].id] = static_cast<int32_t>(i);
  std::vector<sfx_instr> d(ins.size());
  std::vector<TensorValue> vals(ins.size());
  std::vector<void*> ptrs(ins.size());
  for (size_t i = 0; i < ins.size(); ++i) {
    const Instruction& in = ins[i];
    sfx_instr& s = d[i];
    std::memset(&s, 0, sizeof s);
    s.id = in.id.c_str();
    s.opcode = static_cast<int32_t>(in.opcode);
    s.kind = static_cast<int32_t>(in.kind);
    if (in.opcode == Opcode::LibraryCall) s.kind = in.callee == "matmul" ? SFX_CALLEE_MATMUL : SFX_CALLEE_OPAQUE;
    s.dtype = in.shape.etype == ElementType::F32 ? SFX_F32 : SFX_I32;
    s.rank = static_cast<int32_t>(in.shape.rank());
    for (int k = 0; k < s.rank; ++k) s.dims[k] = in.shape.dims[k];
    s.n_operands = static_cast<int32_t>(in.operands.size());
    for (int k = 0; k < s.n_operands && k < 3; ++k) s.operands[k] = index.at(in.operands[k]);
    for (size_t k = 0; k < in.permutation.size(); ++k) s.permutation[k] = in.permutation[k];
    s.n_dim_map = static_cast<int32_t>(in.broadcast_dim_map.size());
    for (size_t k = 0; k < in.broadcast_dim_map.size(); ++k) s.broadcast_dim_map[k] = in.broadcast_dim_map[k];
    s.n_reduce_dims = static_cast<int32_t>(in.reduce_dims.size());
    for (size_t k = 0; k < in.reduce_dims.size(); ++k) s.reduce_dims[k] = in.reduce_dims[k];
    s.reducer = static_cast<int32_t>(in.reducer);
    s.scalar = in.scalar;
    s.n_literal = static_cast<int64_t>(in.literal.size());
    s.literal = in.literal.empty() ? nullptr : in.literal.data();
    vals[i] = in.opcode == Opcode::Parameter ? inputs.at(in.id) : TensorValue::zeros(in.shape);
    ptrs[i] = in.shape.etype == ElementType::F32 ? static_cast<void*>(vals[i].f32.data())
                                                 : static_cast<void*>(vals[i].i32.data());
  }
  sfx_graph_desc gd{};
  gd.n_instrs = static_cast<int32_t>(d.size());
  gd.instrs = d.data();
  if (sfx_oracle_interpret(&gd, ptrs.data(), 1) != 0) throw std::runtime_error(sfx_oracle_error());
  std::map<InstrId, TensorValue> out;
  for (const auto& [id, i] : index) out[id] = vals[i];
  return out;
}

bool reduce_dependent(const TensorGraph& g, const InstrId& id, std::map<InstrId, bool>& memo) {
  auto it = memo.find(id);
  if (it != memo.end()) return it->second;
  bool r = g.at(id).opcode == Opcode::Reduce;
  for (const InstrId& op : g.at(id).operands) r = r || reduce_dependent(g, op, memo);
  return memo[id] = r;
}

int g_via_fp64 = 0;  // outputs accepted by the reduction-order policy

// The reference's own criterion (values_close vs interpret, 1e-5); outputs
// downstream of a reduction may instead meet it against the fp64 restatement
// (reduction-order differences allowed, BASELINE.json north_star).
bool compare(const TensorGraph& g, const std::map<InstrId, TensorValue>& ref, const std::map<InstrId, TensorValue>& dev,
             const std::map<InstrId, TensorValue>& inputs, std::string* why) {
  std::map<InstrId, bool> memo;
  std::map<InstrId, TensorValue> exact;
  // every value of the map (graph outputs and the intermediates the binding
  // reads back from HBM), against interpret's value of that instruction
  for (const auto& [o, v] : dev) {
    if (!ref.count(o)) {
      *why = "unexpected key " + o;
      return false;
    }
    if (testsupport::values_close(v, ref.at(o), 1e-5)) continue;
    if (reduce_dependent(g, o, memo)) {
      if (exact.empty()) exact = interpret_fp64(g, inputs);
      if (testsupport::values_close(dev.at(o), exact.at(o), 1e-5)) {
        ++g_via_fp64;
        continue;
      }
    }
    *why = "value " + o;
    return false;
  }
  return true;
}

// The key set of the reference's run_compiled map (pipeline.cpp:104-118):
// every parameter, constant and unfused instruction, and every group root.
std::set<InstrId> expected_keys(const TensorGraph& g, const CompileReport& report) {
  std::set<InstrId> members, keys;
  for (const CompiledKernel& k : report.kernels) {
    members.insert(k.comp.members.begin(), k.comp.members.end());
    keys.insert(k.comp.roots.begin(), k.comp.roots.end());
  }
  for (const Instruction& i : g.instructions())
    if (!members.count(i.id)) keys.insert(i.id);
  return keys;
}

// On failure with SFX_DUMP_DIR set: the graph, its inputs (parameters in
// instruction order) and both executors' outputs, for offline analysis.
void dump_case(const std::string& name, const TensorGraph& g, const std::map<InstrId, TensorValue>& inputs,
               const std::map<InstrId, TensorValue>& ref, const std::map<InstrId, TensorValue>& dev) {
  const char* dir = std::getenv("SFX_DUMP_DIR");
  if (!dir) return;
  std::string base = std::string(dir) + "/" + name;
  for (char& ch : base)
    if (ch == ' ') ch = '_';
  std::ofstream(base + ".graph.json") << serialize_graph(g);
  auto put = [](std::ofstream& f, const TensorValue& v) {
    if (v.shape.etype == ElementType::F32) f.write(reinterpret_cast<const char*>(v.f32.data()), v.f32.size() * 4);
    else f.write(reinterpret_cast<const char*>(v.i32.data()), v.i32.size() * 4);
  };
  std::ofstream fi(base + ".inputs.bin", std::ios::binary);
  for (const Instruction& i : g.instructions())
    if (i.opcode == Opcode::Parameter) put(fi, inputs.at(i.id));
  std::ofstream fr(base + ".ref.bin", std::ios::binary), fd(base + ".dev.bin", std::ios::binary);
  for (const InstrId& o : g.outputs()) {
    put(fr, ref.at(o));
    if (dev.count(o)) put(fd, dev.at(o));
  }
}

void run_case(const std::string& name, const TensorGraph& g, const CompileReport& report,
              const std::map<InstrId, TensorValue>& inputs, Tally& t) {
  ++t.cases;
  try {
    auto ref = interpret(g, inputs);
    long long before = stitchfuse_device::launches();
    auto dev = stitchfuse_device::run_compiled(report, g, inputs);
    long long launched = stitchfuse_device::launches() - before;
    std::string why;
    if (launched != expected_launches(report)) {
      t.fail(name + ": launched " + std::to_string(launched) + " kernels for " +
             std::to_string(report.kernels.size()) + " fused groups + " +
             std::to_string(report.fusion.unfused.size()) + " unfused instructions");
    } else if ([&] {
                 std::set<InstrId> got;
                 for (const auto& kv : dev) got.insert(kv.first);
                 return got != expected_keys(g, report);
               }()) {
      t.fail(name + ": run_compiled map keys differ from the reference's");
    } else if (!compare(g, ref, dev, inputs, &why)) {
      t.fail(name + ": " + why);
      dump_case(name, g, inputs, ref, dev);
    } else {
      ++t.passed;
    }
  } catch (const std::exception& e) {
    t.fail(name + ": " + e.what());
  }
}

int finish(const std::string& mode, const Tally& t, int extra_skipped) {
  json line = {{"mode", mode}, {"cases", t.cases}, {"passed", t.passed}, {"skipped_ineligible", extra_skipped},
               {"outputs_accepted_vs_fp64", g_via_fp64}, {"failures", t.failures}};
  std::cout << line.dump() << std::endl;
  return t.cases > 0 && t.passed == t.cases ? 0 : 1;
}

int cmd_random(uint64_t seed, int count, bool alternate) {
  std::mt19937_64 rng(seed);
  testsupport::RandomGraphConfig cfg;
  Tally t;
  int skipped = 0;
  for (int i = 0; i < count; ++i) {
    TensorGraph g = testsupport::random_graph(rng, cfg);
    PipelineOptions o;
    o.fuse_dot = alternate && (i % 2 == 0);  // test_acceptance.cpp:48, test_pipeline.cpp:111
    PerfLibrary lib;
    CostModelParams params;
    CompileReport report = compile_graph(g, o, lib, params);
    auto inputs = testsupport::random_inputs(g, rng);  // same rng stream as test_acceptance.cpp:50-53
    if (!eligible(g)) {
      ++skipped;
      continue;
    }
    run_case("graph " + std::to_string(i), g, report, inputs, t);
  }
  return finish("random seed " + std::to_string(seed), t, skipped);
}

int cmd_schedules() {
  Tally t;
  int skipped = 0;
  for (const auto& [name, text] : fixture_graphs()) {
    TensorGraph g = parse_graph(text);
    if (!eligible(g)) {
      ++skipped;
      continue;
    }
    PipelineOptions options;
    SpanMap sm = compute_span(g);
    FusionPlan fusion = fuse_module(g, options);
    std::mt19937_64 rng(101);
    auto inputs = testsupport::random_inputs(g, rng);
    auto reference = interpret(g, inputs);
    for (const FusedComputation& comp : fusion.computations) {
      if (comp.roots.size() != 1) continue;
      const InstrId& root = comp.roots[0];
      for (const Schedule& sched : enumerate_schedules(g.at(root).shape)) {
        ResolveResult r = resolve_schedule(comp, g, {{root, sched}}, options);
        if (!r.ok()) continue;
        SmemResult smem = plan_shared_memory(comp, g, sm, *r.plan, options);
        if (!std::holds_alternative<SharedMemPlan>(smem)) continue;
        KernelProgram program = emit_program(comp, g, sm, *r.plan, std::get<SharedMemPlan>(smem), options);
        if (check_program(program, g)) continue;
        std::map<InstrId, TensorValue> externals;
        for (const InstrId& id : comp.members)
          for (const InstrId& op : g.at(id).operands)
            if (!comp.members.count(op)) externals[op] = reference.at(op);
        ++t.cases;
        std::string label = name + " " + root + " " + to_string(sched);
        try {
          auto outs = stitchfuse_device::run_program(program, g, externals);
          bool ok = true;
          for (size_t k = 0; k < comp.roots.size(); ++k)
            ok = ok && testsupport::values_close(outs[k], reference.at(comp.roots[k]), 1e-5);
          if (ok) ++t.passed;
          else t.fail(label);
        } catch (const std::exception& e) {
          t.fail(label + ": " + e.what());
        }
      }
    }
  }
  return finish("schedules", t, skipped);
}

int cmd_shrink(uint64_t seed, int count) {
  Tally t;
  int skipped = 0;
  std::mt19937_64 rng(seed);
  testsupport::RandomGraphConfig cfg;
  cfg.allow_library_calls = false;
  std::vector<std::pair<std::string, TensorGraph>> graphs;
  for (const auto& [name, text] : fixture_graphs()) graphs.push_back({name, parse_graph(text)});
  for (int i = 0; i < count; ++i) graphs.push_back({"random " + std::to_string(i), testsupport::random_graph(rng, cfg)});
  for (const auto& [name, g] : graphs) {
    if (!eligible(g)) {
      ++skipped;
      continue;
    }
    std::mt19937_64 irng(103);
    auto inputs = testsupport::random_inputs(g, irng);
    for (int64_t limit : {20480, 1024, 256}) {
      PipelineOptions options;
      options.smem_limit = limit;
      PerfLibrary lib;
      CostModelParams params;
      CompileReport report;
      try {
        report = compile_graph(g, options, lib, params);
      } catch (const std::exception&) {
        continue;  // planner cannot meet this limit
      }
      run_case(name + " smem_limit " + std::to_string(limit), g, report, inputs, t);
    }
  }
  return finish("shrink", t, skipped);
}

// Acceptance criterion 9 (test_acceptance.cpp:375-391): 50 random fuse_dot
// plans (rng 90001) executed with full coverage — here with the device
// coverage check around every launch (debug_checks=1) — and, beyond the
// reference's criterion, compared with its interpret.
int cmd_crit9() {
  Tally t;
  int skipped = 0;
  CostModelParams params;
  std::mt19937_64 rng2(90001);
  stitchfuse_device::set_debug_checks(1);
  for (int i = 0; i < 50; ++i) {
    TensorGraph g = testsupport::random_graph(rng2);
    PipelineOptions options;
    options.fuse_dot = true;
    PerfLibrary lib;
    CompileReport rep;
    try {
      rep = compile_graph(g, options, lib, params);
    } catch (const std::exception& e) {
      ++t.cases;
      t.fail("graph " + std::to_string(i) + ": compile_graph: " + e.what());
      continue;
    }
    auto inputs = testsupport::random_inputs(g, rng2);  // same rng order as the reference test
    if (!eligible(g)) {
      ++skipped;
      continue;
    }
    run_case("graph " + std::to_string(i), g, rep, inputs, t);
  }
  stitchfuse_device::set_debug_checks(0);
  return finish("criterion 9 (fuse_dot, coverage-checked)", t, skipped);
}

// Acceptance criterion 7's executor leg (test_acceptance.cpp:291-312): the
// fuse_dot fixture planned under smem_limit 1024 (shrunk [Exponential.1,
// Divide.1]) keeps Dot.1 values_close to interpret.
int cmd_crit7() {
  Tally t;
  TensorGraph g = parse_graph(fixture_graphs().at("softmax_batchdot"));  // test_acceptance.cpp:29
  PipelineOptions options;
  options.fuse_dot = true;
  options.smem_limit = 1024;
  PerfLibrary lib;
  CostModelParams params;
  CompileReport rep = compile_graph(g, options, lib, params);
  std::mt19937_64 rng2(70001);
  auto inputs = testsupport::random_inputs(g, rng2);
  ++t.cases;
  try {
    auto ref = interpret(g, inputs);
    auto dev = stitchfuse_device::run_compiled(rep, g, inputs);
    if (rep.kernels[0].smem.shrunk != std::vector<InstrId>{"Exponential.1", "Divide.1"}) t.fail("shrink order");
    else if (!testsupport::values_close(dev.at("Dot.1"), ref.at("Dot.1"), 1e-5)) t.fail("Dot.1");
    else ++t.passed;
  } catch (const std::exception& e) {
    t.fail(e.what());
  }
  return finish("criterion 7 (shrunk fuse_dot fixture)", t, 0);
}

// The binding caches compiled plans by signature: repeated run_compiled /
// run_program calls on one plan compile once, launch every time, and return
// the same values; a different plan compiles again.
int cmd_cache() {
  Tally t;
  std::mt19937_64 rng(113);
  testsupport::RandomGraphConfig cfg;
  cfg.allow_library_calls = false;
  TensorGraph g = testsupport::random_graph(rng, cfg);
  TensorGraph g2 = testsupport::random_graph(rng, cfg);
  PipelineOptions o;
  PerfLibrary lib;
  CostModelParams params;
  CompileReport rep = compile_graph(g, o, lib, params);
  CompileReport rep2 = compile_graph(g2, o, lib, params);
  auto inputs = testsupport::random_inputs(g, rng);
  auto inputs2 = testsupport::random_inputs(g2, rng);
  auto ref = interpret(g, inputs);
  auto check_round = [&](const std::string& what, long long want_compiles) {
    ++t.cases;
    long long c0 = stitchfuse_device::compiles(), l0 = stitchfuse_device::launches();
    auto dev = stitchfuse_device::run_compiled(rep, g, inputs);
    long long dc = stitchfuse_device::compiles() - c0, dl = stitchfuse_device::launches() - l0;
    std::string why;
    if (dc != want_compiles) t.fail(what + ": " + std::to_string(dc) + " compiles");
    else if (dl != expected_launches(rep)) t.fail(what + ": " + std::to_string(dl) + " launches");
    else if (!compare(g, ref, dev, inputs, &why)) t.fail(what + ": " + why);
    else ++t.passed;
  };
  check_round("first run_compiled", 1);
  check_round("second run_compiled", 0);
  ++t.cases;
  long long c0 = stitchfuse_device::compiles();
  stitchfuse_device::run_compiled(rep2, g2, inputs2);
  if (stitchfuse_device::compiles() - c0 == 1) ++t.passed;
  else t.fail("a different plan must compile");
  check_round("back to the first plan", 0);
  // run_program: one group, twice
  const KernelProgram& prog = rep.kernels.at(0).program;
  std::map<InstrId, TensorValue> ext;
  for (const InstrId& id : prog.comp.members)
    for (const InstrId& op : g.at(id).operands)
      if (!prog.comp.members.count(op)) ext[op] = ref.at(op);
  for (int r = 0; r < 2; ++r) {
    ++t.cases;
    long long k0 = stitchfuse_device::compiles();
    auto outs = stitchfuse_device::run_program(prog, g, ext);
    bool ok = stitchfuse_device::compiles() - k0 == (r == 0 ? 1 : 0);
    for (size_t k = 0; k < prog.comp.roots.size(); ++k)
      ok = ok && testsupport::values_close(outs[k], ref.at(prog.comp.roots[k]), 1e-5);
    if (ok) ++t.passed;
    else t.fail("run_program round " + std::to_string(r));
  }
  return finish("binding cache", t, 0);
}

// The executor self-checks: each corrupted program (the reference's own two
// from test_exec.cpp:157-194, plus an overlapping root write and a containment
// violation) must make both run_program implementations throw ExecError, and
// the device binding's message must carry the reference's.
int cmd_selfchecks() {
  Tally t;
  CostModelParams params;
  auto plan = [&](const std::string& fixture, bool fuse_dot) {
    PipelineOptions o;
    o.fuse_dot = fuse_dot;
    PerfLibrary lib;
    TensorGraph g = parse_graph(fixture_graphs().at(fixture));
    return std::make_pair(g, compile_graph(g, o, lib, params));
  };
  auto expect = [&](const std::string& name, const TensorGraph& g, const KernelProgram& prog, uint64_t seed) {
    ++t.cases;
    std::mt19937_64 rng(seed);
    auto inputs = testsupport::random_inputs(g, rng);
    std::map<InstrId, TensorValue> ext;
    for (const InstrId& m : prog.comp.members)
      for (const InstrId& op : g.at(m).operands)
        if (!prog.comp.members.count(op)) ext[op] = inputs.count(op) ? inputs.at(op) : constant_value(g.at(op));
    std::string ref_msg, dev_msg;
    try {
      run_program(prog, g, ext);
    } catch (const ExecError& e) {
      ref_msg = e.what();
    }
    try {
      stitchfuse_device::run_program(prog, g, ext);
    } catch (const ExecError& e) {
      dev_msg = e.what();
    }
    if (ref_msg.empty()) t.fail(name + ": the reference did not throw");
    else if (dev_msg.find(ref_msg) == std::string::npos) t.fail(name + ": reference '" + ref_msg + "', device '" + dev_msg + "'");
    else ++t.passed;
  };
  {
    auto [g, rep] = plan("softmax_batchdot", true);
    KernelProgram p = rep.kernels[0].program;
    for (Statement& st : p.statements)  // test_exec.cpp:165-169
      if (auto* mat = std::get_if<MaterializeStmt>(&st))
        if (auto* sh = std::get_if<SharedDest>(&mat->dest))
          if (mat->instr == "Reduce.1" || mat->instr == "Reduce.2") sh->offset = 0;
    expect("stale arena read", g, p, 105);
    KernelProgram q = rep.kernels[0].program;
    q.plan.per_instruction.at("Exponential.1").sword *= 2;
    expect("chunk containment", g, q, 105);
  }
  {
    auto [g, rep] = plan("elementwise_chain", false);
    KernelProgram p = rep.kernels[0].program;
    for (Statement& st : p.statements)  // test_exec.cpp:183-187
      if (auto* mat = std::get_if<MaterializeStmt>(&st))
        if (std::holds_alternative<OutputDest>(mat->dest) && mat->schedule.sword > 1) mat->schedule.sword *= 2;
    expect("incomplete coverage", g, p, 107);
    KernelProgram q = rep.kernels[0].program;
    for (Statement& st : q.statements)
      if (auto* mat = std::get_if<MaterializeStmt>(&st))
        if (std::holds_alternative<OutputDest>(mat->dest)) mat->schedule.sword /= 2;
    expect("overlapping root write", g, q, 107);
  }
  return finish("executor self-checks", t, 0);
}

std::vector<std::pair<InstrId, std::set<InstrId>>> membership(const CompileReport& r) {
  std::vector<std::pair<InstrId, std::set<InstrId>>> m;
  for (const CompiledKernel& k : r.kernels) m.push_back({k.comp.fusion_root, k.comp.members});
  return m;
}

// The measured perf library (integration/): plan a graph, measure every key
// the planner missed on the device (literal tier under that key's schedule),
// re-plan with the measured library (no misses left), then tune the planned
// groups' template parameters on miss.  Default-library plans are the parity
// contract: their membership is printed next to the measured one.
int cmd_perflib(const std::string& graph_path, const std::string& lib_out, const std::string& tp_out, int max_keys) {
  std::ifstream in(graph_path);
  std::stringstream ss;
  ss << in.rdbuf();
  TensorGraph g = parse_graph(ss.str());
  PipelineOptions o;
  CostModelParams params;
  PerfLibrary empty;
  CompileReport base = compile_graph(g, o, empty, params);
  PerfLibrary lib;
  auto t0 = std::chrono::steady_clock::now();
  stitchfuse_device::MeasureStats ms = stitchfuse_device::measure_misses(g, o, lib, params, 10, max_keys);
  double measure_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  size_t measured = 0;
  for (const auto& [k, e] : lib.entries()) measured += !e.synthetic;
  lib.hits_ = lib.misses_ = 0;
  PerfLibrary replan = lib;
  CompileReport with = compile_graph(g, o, replan, params);
  stitchfuse_device::MeasureStats tt = stitchfuse_device::tune_templates(base, g, 20);
  stitchfuse_device::MeasureStats again = stitchfuse_device::tune_templates(base, g, 20);
  lib.store(lib_out);
  std::ofstream(tp_out) << stitchfuse_device::template_params_text();
  json line = {{"mode", "perflib"}, {"graph", graph_path}, {"keys_missed", ms.keys_missed},
               {"keys_measured", ms.keys_measured}, {"measured_entries", measured}, {"measure_seconds", measure_s},
               {"replan_misses", replan.misses()}, {"replan_hits", replan.hits()},
               {"membership_default_equals_measured", membership(base) == membership(with)},
               {"groups_default", base.kernels.size()}, {"groups_measured", with.kernels.size()},
               {"groups_tuned", tt.groups_tuned}, {"groups_changed", tt.groups_changed},
               {"retune_groups_tuned", again.groups_tuned}, {"notes", tt.notes}, {"measure_notes", ms.notes}};
  std::cout << line.dump() << std::endl;
  const bool ok = ms.keys_measured > 0 && replan.misses() == 0 && tt.groups_tuned > 0 && again.groups_tuned == 0;
  return ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::runtime_error("usage: device_parity random|schedules|shrink ...");
    std::vector<std::string> pos;
    bool alt = false;
    for (int i = 1; i < argc; ++i) {
      if (!std::strcmp(argv[i], "--literal")) stitchfuse_device::set_strategy(SFX_STRATEGY_LITERAL);
      else if (!std::strcmp(argv[i], "--fuse-dot-alternate")) alt = true;
      else pos.push_back(argv[i]);
    }
    std::string cmd = pos.at(0);
    if (cmd == "random") return cmd_random(std::stoull(pos.at(1)), std::stoi(pos.at(2)), alt);
    if (cmd == "schedules") return cmd_schedules();
    if (cmd == "crit9") return cmd_crit9();
    if (cmd == "crit7") return cmd_crit7();
    if (cmd == "cache") return cmd_cache();
    if (cmd == "selfchecks") return cmd_selfchecks();
    if (cmd == "perflib")
      return cmd_perflib(pos.at(1), pos.at(2), pos.at(3), pos.size() > 4 ? std::stoi(pos[4]) : -1);
    if (cmd == "shrink") return cmd_shrink(pos.size() > 1 ? std::stoull(pos[1]) : 7, pos.size() > 2 ? std::stoi(pos[2]) : 30);
    throw std::runtime_error("unknown command " + cmd);
  } catch (const std::exception& e) {
    std::cerr << "device_parity error: " << e.what() << "\n";
    return 2;
  }
}
