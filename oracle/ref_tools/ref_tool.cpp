// TEST INFRASTRUCTURE — reference-side tool, linked against the reference
// library compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/.  It is the only way this repo touches the reference planner and
// executor: it exports the reference's own fusion plans (compile_graph,
// pipeline.cpp:18-63) and the reference's own outputs (interpret,
// exec.cpp:249-268; run_compiled, pipeline.cpp:65-133) so the tests can pin the
// oracle restatement and the device executor against them.  Nothing in the
// product (paper_1811_05213_b200/) links or calls this.
//
//   ref_tool plan   <graph.json> [--fuse-dot] [--smem-limit N] [--footprint-limit N]
//                                                                   -> plan bundle JSON (stdout)
//   ref_tool random <seed> <count> <outdir> [--no-libcalls] [--fuse-dot-alternate]
//                                                                   -> one bundle per graph
//   ref_tool run    <bundle-or-graph.json> <seed> <lo> <hi> <out-prefix> [--compiled] [--no-interpret]
//                                                                   -> <prefix>.interpret.bin / .compiled.bin
//   ref_tool bench  <graph.json> <seed> <threads> <iters> [--interpret] [--footprint-limit N]
//                                                                   -> JSON timing line
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <thread>

#include "json.hpp"
#include "stitchfuse/exec.hpp"
#include "stitchfuse/fixtures.hpp"
#include "stitchfuse/pipeline.hpp"
#include "support.hpp"

extern "C" {
#include "../sfx_gen.h"
}

using namespace stitchfuse;
using json = nlohmann::json;

namespace {

std::string slurp(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot read " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

const char* sched_name(SchedType t) { return t == SchedType::Row ? "row" : "col"; }

json schedule_json(const Schedule& s) { return json::array({s.split_dim, s.sword, sched_name(s.type)}); }

json report_json(const CompileReport& report, const TensorGraph& graph, const PipelineOptions& o) {
  json doc;
  doc["graph"] = json::parse(serialize_graph(graph));
  doc["options"] = {{"fuse_dot", o.fuse_dot},
                    {"footprint_limit", o.footprint_limit},
                    {"smem_limit", o.smem_limit}};
  doc["baseline_kernels"] = report.baseline_kernels;
  doc["fused_kernels"] = report.fused_kernels;
  doc["fusion_ratio"] = report.fusion_ratio;
  doc["unfused"] = std::vector<std::string>(report.fusion.unfused.begin(), report.fusion.unfused.end());
  json kernels = json::array();
  for (const CompiledKernel& k : report.kernels) {
    json jk;
    jk["fusion_root"] = k.comp.fusion_root;
    jk["members"] = std::vector<std::string>(k.comp.members.begin(), k.comp.members.end());
    jk["roots"] = k.comp.roots;
    jk["footprint_bytes"] = k.comp.footprint_bytes;
    jk["blocks"] = k.plan.blocks;
    jk["block_threads"] = k.plan.block_threads;
    jk["bypassed"] = std::vector<std::string>(k.plan.bypassed.begin(), k.plan.bypassed.end());
    json per = json::object();
    for (const auto& [id, s] : k.plan.per_instruction) per[id] = schedule_json(s);
    jk["per_instruction"] = per;
    jk["arena_bytes"] = k.program.arena_bytes;
    json offs = json::object();
    for (const auto& [id, off] : k.program.arena_offsets) offs[id] = off;
    jk["arena_offsets"] = offs;
    jk["smem_total_bytes"] = k.smem.total_bytes;
    jk["shrunk"] = k.smem.shrunk;
    json stmts = json::array();
    for (const Statement& st : k.program.statements) {
      json js;
      if (const auto* m = std::get_if<MaterializeStmt>(&st)) {
        js["kind"] = "materialize";
        js["instr"] = m->instr;
        js["schedule"] = schedule_json(m->schedule);
        if (const auto* sh = std::get_if<SharedDest>(&m->dest)) {
          js["dest"] = "shared";
          js["offset"] = sh->offset;
          js["bytes"] = sh->bytes;
        } else {
          js["dest"] = "output";
          js["root_index"] = std::get<OutputDest>(m->dest).root_index;
        }
      } else if (std::holds_alternative<BarrierStmt>(st)) {
        js["kind"] = "barrier";
      } else {
        js["kind"] = "inline";
        js["instr"] = std::get<InlineBindingStmt>(st).instr;
      }
      stmts.push_back(js);
    }
    jk["statements"] = stmts;
    jk["cost_us"] = k.cost_us;
    jk["dump"] = dump_program(k.program, graph);
    kernels.push_back(jk);
  }
  doc["kernels"] = kernels;
  return doc;
}

CompileReport compile(const TensorGraph& g, const PipelineOptions& o) {
  PerfLibrary lib;
  CostModelParams params;
  return compile_graph(g, o, lib, params);
}

bool device_eligible(const TensorGraph& g, const CompileReport& r) {
  // everything the reference can execute: "opaque" library calls are
  // barriers only (exec.cpp:207-209)
  for (const Instruction& i : g.instructions())
    if (i.opcode == Opcode::LibraryCall && i.callee != "matmul") return false;
  (void)r;
  return true;
}

std::map<InstrId, TensorValue> gen_inputs(const TensorGraph& g, uint64_t seed, float lo, float hi) {
  std::map<InstrId, TensorValue> inputs;
  uint64_t t = 0;
  for (const Instruction& instr : g.instructions()) {
    if (instr.opcode != Opcode::Parameter) continue;
    TensorValue v = TensorValue::zeros(instr.shape);
    if (instr.shape.etype == ElementType::F32)
      sfx_gen_f32(seed, t, lo, hi, v.f32.data(), instr.shape.element_count());
    else
      sfx_gen_i32(seed, t, v.i32.data(), instr.shape.element_count());
    inputs[instr.id] = std::move(v);
    ++t;
  }
  return inputs;
}

TensorGraph load_any(const std::string& path) {
  json doc = json::parse(slurp(path));
  if (doc.contains("graph")) return parse_graph(doc["graph"].dump());
  return parse_graph(doc.dump());
}

void write_outputs(const std::string& path, const TensorGraph& g,
                   const std::map<InstrId, TensorValue>& values) {
  std::ofstream out(path, std::ios::binary);
  for (const InstrId& id : g.outputs()) {
    const TensorValue& v = values.at(id);
    if (v.shape.etype == ElementType::F32)
      out.write(reinterpret_cast<const char*>(v.f32.data()), v.f32.size() * 4);
    else
      out.write(reinterpret_cast<const char*>(v.i32.data()), v.i32.size() * 4);
  }
}

uint64_t fnv1a(const std::map<InstrId, TensorValue>& values, const TensorGraph& g) {
  uint64_t h = 1469598103934665603ull;
  for (const InstrId& id : g.outputs()) {
    const TensorValue& v = values.at(id);
    const unsigned char* p = v.shape.etype == ElementType::F32
                                 ? reinterpret_cast<const unsigned char*>(v.f32.data())
                                 : reinterpret_cast<const unsigned char*>(v.i32.data());
    size_t n = v.shape.element_count() * 4;
    for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  }
  return h;
}

int cmd_plan(int argc, char** argv) {
  if (argc < 3) throw std::runtime_error("usage: plan <graph.json> [--fuse-dot] [--smem-limit N]");
  PipelineOptions o;
  for (int i = 3; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--fuse-dot")) o.fuse_dot = true;
    else if (!std::strcmp(argv[i], "--smem-limit") && i + 1 < argc) o.smem_limit = std::stoll(argv[++i]);
    else if (!std::strcmp(argv[i], "--footprint-limit") && i + 1 < argc) o.footprint_limit = std::stoll(argv[++i]);
  }
  TensorGraph g = parse_graph(slurp(argv[2]));
  CompileReport r = compile(g, o);
  std::cout << report_json(r, g, o).dump(1) << "\n";
  return 0;
}

int cmd_random(int argc, char** argv) {
  if (argc < 5) throw std::runtime_error("usage: random <seed> <count> <outdir> [flags]");
  uint64_t seed = std::stoull(argv[2]);
  int count = std::stoi(argv[3]);
  std::string outdir = argv[4];
  bool no_lib = false, alternate = false, device_only = false;
  for (int i = 5; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--no-libcalls")) no_lib = true;
    if (!std::strcmp(argv[i], "--fuse-dot-alternate")) alternate = true;
    if (!std::strcmp(argv[i], "--device-only")) device_only = true;
  }
  std::mt19937_64 rng(seed);
  testsupport::RandomGraphConfig cfg;
  cfg.allow_library_calls = !no_lib;
  int written = 0;
  for (int i = 0; i < count; ++i) {
    TensorGraph g = testsupport::random_graph(rng, cfg);
    PipelineOptions o;
    o.fuse_dot = alternate && (i % 2 == 0);  // test_acceptance.cpp:48, test_pipeline.cpp:111
    CompileReport r = compile(g, o);
    bool elig = device_eligible(g, r);
    if (device_only && !elig) continue;
    json doc = report_json(r, g, o);
    doc["stream"] = {{"seed", seed}, {"index", i}, {"device_eligible", elig}};
    char name[256];
    std::snprintf(name, sizeof name, "%s/rand_s%llu_%03d.json", outdir.c_str(),
                  static_cast<unsigned long long>(seed), i);
    std::ofstream(name) << doc.dump() << "\n";
    ++written;
  }
  std::cout << written << "\n";
  return 0;
}

int cmd_run(int argc, char** argv) {
  if (argc < 7) throw std::runtime_error("usage: run <graph> <seed> <lo> <hi> <out-prefix> [--compiled]");
  TensorGraph g = load_any(argv[2]);
  uint64_t seed = std::stoull(argv[3]);
  float lo = std::stof(argv[4]), hi = std::stof(argv[5]);
  std::string prefix = argv[6];
  bool compiled = false, interp = true;
  for (int i = 7; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--compiled")) compiled = true;
    if (!std::strcmp(argv[i], "--no-interpret")) interp = false;
  }
  auto inputs = gen_inputs(g, seed, lo, hi);
  json line;
  if (interp) {
    auto t0 = std::chrono::steady_clock::now();
    auto v = interpret(g, inputs);
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    write_outputs(prefix + ".interpret.bin", g, v);
    line["interpret_s"] = s;
    line["interpret_fnv"] = fnv1a(v, g);
  }
  if (compiled) {
    PipelineOptions o;
    CompileReport r = compile(g, o);
    auto t0 = std::chrono::steady_clock::now();
    auto v = run_compiled(r, g, inputs);
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    write_outputs(prefix + ".compiled.bin", g, v);
    line["compiled_s"] = s;
    line["compiled_fnv"] = fnv1a(v, g);
  }
  std::cout << line.dump() << "\n";
  return 0;
}

// Times the reference executor on `threads` independent instances (it is
// single-threaded and reentrant); each thread compiles its own
// plan and runs run_compiled (or interpret) `iters` times.
int cmd_bench(int argc, char** argv) {
  if (argc < 6)
    throw std::runtime_error("usage: bench <graph> <seed> <threads> <iters> [--interpret] [--footprint-limit N]");
  TensorGraph g = load_any(argv[2]);
  uint64_t seed = std::stoull(argv[3]);
  int threads = std::stoi(argv[4]);
  int iters = std::stoi(argv[5]);
  bool use_interp = false;
  PipelineOptions o;
  for (int i = 6; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--interpret")) use_interp = true;
    else if (!std::strcmp(argv[i], "--footprint-limit") && i + 1 < argc) o.footprint_limit = std::stoll(argv[++i]);
  }
  auto inputs = gen_inputs(g, seed, -1.0f, 1.0f);
  CompileReport r = compile(g, o);
  std::atomic<uint64_t> sink{0};
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&]() {
      for (int i = 0; i < iters; ++i) {
        auto v = use_interp ? interpret(g, inputs) : run_compiled(r, g, inputs);
        sink += v.size();
      }
    });
  for (auto& th : pool) th.join();
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  json groups = json::array();
  for (const auto& k : r.kernels) groups.push_back(k.comp.fusion_root);
  json line = {{"seconds", s}, {"threads", threads}, {"iters", iters},
               {"executor", use_interp ? "interpret" : "run_compiled"},
               {"fused_kernels", r.fused_kernels}, {"groups", groups}, {"footprint_limit", o.footprint_limit}};
  std::cout << line.dump() << "\n";
  return sink.load() > 0 ? 0 : 1;
}

// Loads a (measured) performance library with the reference's own parser
// (PerfLibrary::load, tuning.cpp:41-90) and plans the graph with it.
int cmd_perflib(int argc, char** argv) {
  if (argc < 4) throw std::runtime_error("usage: perflib <graph> <perf.lib>");
  TensorGraph g = load_any(argv[2]);
  PerfLibrary lib = PerfLibrary::load(argv[3]);
  size_t measured = 0;
  for (const auto& [k, e] : lib.entries())
    if (!e.synthetic) ++measured;
  PipelineOptions o;
  CostModelParams params;
  CompileReport with = compile_graph(g, o, lib, params);
  PerfLibrary empty;
  CompileReport base = compile_graph(g, o, empty, params);
  json line = {{"entries", lib.entries().size()}, {"measured_entries", measured}, {"hits", lib.hits()},
               {"misses", lib.misses()}, {"fused_kernels", with.fused_kernels},
               {"fused_kernels_default", base.fused_kernels}};
  json kernels = json::array();
  for (size_t i = 0; i < with.kernels.size(); ++i)
    kernels.push_back({{"fusion_root", with.kernels[i].comp.fusion_root}, {"cost_us", with.kernels[i].cost_us},
                       {"members", with.kernels[i].comp.members.size()},
                       {"same_members_as_default", i < base.kernels.size() &&
                                                       base.kernels[i].comp.members == with.kernels[i].comp.members}});
  line["kernels"] = kernels;
  std::cout << line.dump() << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::runtime_error("usage: ref_tool plan|random|run|bench ...");
    std::string cmd = argv[1];
    if (cmd == "plan") return cmd_plan(argc, argv);
    if (cmd == "random") return cmd_random(argc, argv);
    if (cmd == "run") return cmd_run(argc, argv);
    if (cmd == "bench") return cmd_bench(argc, argv);
    if (cmd == "perflib") return cmd_perflib(argc, argv);
    if (cmd == "fixture") {
      std::cout << fixture_graphs().at(argv[2]);
      return 0;
    }
    throw std::runtime_error("unknown command " + cmd);
  } catch (const std::exception& e) {
    std::cerr << "ref_tool error: " << e.what() << "\n";
    return 2;
  }
}
