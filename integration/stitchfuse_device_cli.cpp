// stitchfuse-device: the reference CLI's `run` command with the B200 executor.
//
//   stitchfuse-device [global flags] run <graph.json> --inputs <tensors.json>
//                     [--compare-reference] [--dump-values] [--host] [--literal]
//   global flags (before or after the command): --fuse-dot --footprint-limit N
//     --smem-limit N --perf-lib PATH --cost-params PATH --seed N
//
// Same inputs file, plan, output lines and exit codes as the reference's
// `stitchfuse run` (reference proj/tools/stitchfuse.cpp:52-88 inputs,
// :122-171 flags, :231-261 run): the graph is parsed and planned by the
// reference's own parse_graph / compile_graph, then executed by
// stitchfuse_device::run_compiled (one sm_100a launch per fusion group) instead
// of stitchfuse::run_compiled; --compare-reference checks against the
// reference's interpret.  --host runs the reference executor instead (A/B).
// Exit codes: 0 success, 1 user error, 2 internal error or reference mismatch.
//
// Built by oracle/Makefile (target `cli`) against the reference library compiled
// from /root/reference; the reference's CLI itself needs CLI11, which is absent.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "json.hpp"
#include "sfx.h"
#include "stitchfuse/exec.hpp"
#include "stitchfuse/pipeline.hpp"
#include "stitchfuse_device.hpp"

using nlohmann::json;
using namespace stitchfuse;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw UsageError("cannot open " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// Tensors file: {id: {"shape": [...], "dtype": "f32"|"i32", "data": [...]}} or
// {"random_seed": s} (default: --seed) — mt19937_64 with
// uniform_real_distribution<float>(-1, 1) / uniform_int_distribution<int32_t>(-4, 4).
std::map<InstrId, TensorValue> read_inputs(const std::string& path, const TensorGraph& g, uint64_t seed) {
  json doc;
  try {
    doc = json::parse(read_file(path));
  } catch (const json::parse_error& e) {
    throw UsageError(path + ": " + e.what());
  }
  std::map<InstrId, TensorValue> out;
  for (const auto& [id, spec] : doc.items()) {
    Shape sh;
    sh.dims = spec.at("shape").get<std::vector<int64_t>>();
    const bool i32 = spec.value("dtype", std::string("f32")) == "i32";
    sh.etype = i32 ? ElementType::I32 : ElementType::F32;
    TensorValue v = TensorValue::zeros(sh);
    const int64_t n = sh.element_count();
    if (spec.contains("data")) {
      const auto data = spec["data"].get<std::vector<double>>();
      if (static_cast<int64_t>(data.size()) != n) throw UsageError(path + ": " + id + ": data size mismatch");
      for (int64_t i = 0; i < n; ++i) {
        if (i32) v.i32[i] = static_cast<int32_t>(data[i]);
        else v.f32[i] = static_cast<float>(data[i]);
      }
    } else {
      std::mt19937_64 gen(spec.value("random_seed", seed));
      std::uniform_real_distribution<float> uf(-1.0f, 1.0f);
      std::uniform_int_distribution<int32_t> ui(-4, 4);
      for (int64_t i = 0; i < n; ++i) {
        if (i32) v.i32[i] = ui(gen);
        else v.f32[i] = uf(gen);
      }
    }
    if (!g.contains(id)) throw UsageError(path + ": unknown input id " + id);
    out[id] = std::move(v);
  }
  return out;
}

double checksum(const TensorValue& v) {
  double s = 0.0;
  if (v.shape.etype == ElementType::F32)
    for (float x : v.f32) s += x;
  else
    for (int32_t x : v.i32) s += x;
  return s;
}

// The CLI's comparison (no NaN special case, as in the reference CLI).
bool close_enough(const TensorValue& a, const TensorValue& b, double rel) {
  if (a.shape != b.shape) return false;
  if (a.shape.etype == ElementType::I32) return a.i32 == b.i32;
  for (size_t i = 0; i < a.f32.size(); ++i) {
    const double x = a.f32[i], y = b.f32[i];
    if (std::abs(x - y) > rel * std::max({1.0, std::abs(x), std::abs(y)})) return false;
  }
  return true;
}

struct Args {
  PipelineOptions options;
  std::string perf_lib, cost_params, command, graph, inputs;
  bool compare = false, dump = false, host = false, literal = false;
};

Args parse_args(int argc, char** argv) {
  Args a;
  std::vector<std::string> pos;
  auto need = [&](int& i) -> std::string {
    if (i + 1 >= argc) throw UsageError(std::string(argv[i]) + " needs a value");
    return argv[++i];
  };
  for (int i = 1; i < argc; ++i) {
    std::string s = argv[i];
    try {
      if (s == "--fuse-dot") a.options.fuse_dot = true;
      else if (s == "--footprint-limit") a.options.footprint_limit = std::stoll(need(i));
      else if (s == "--smem-limit") a.options.smem_limit = std::stoll(need(i));
      else if (s == "--perf-lib") a.perf_lib = need(i);
      else if (s == "--cost-params") a.cost_params = need(i);
      else if (s == "--seed") a.options.seed = std::stoull(need(i));
      else if (s == "--inputs") a.inputs = need(i);
      else if (s == "--compare-reference") a.compare = true;
      else if (s == "--dump-values") a.dump = true;
      else if (s == "--host") a.host = true;
      else if (s == "--literal") a.literal = true;
      else if (s.rfind("--", 0) == 0) throw UsageError("unknown option " + s);
      else pos.push_back(s);
    } catch (const std::logic_error& e) {
      if (dynamic_cast<const UsageError*>(&e)) throw;
      throw UsageError("bad value for " + s);
    }
  }
  if (pos.empty()) throw UsageError("a command is required: run");
  a.command = pos[0];
  if (a.command != "run") throw UsageError("unknown command " + a.command + " (this tool implements run)");
  if (pos.size() != 2) throw UsageError("run: expected one graph file");
  a.graph = pos[1];
  if (a.inputs.empty()) throw UsageError("run: --inputs is required");
  return a;
}

int run(const Args& a) {
  CostModelParams params;
  if (!a.cost_params.empty()) params = CostModelParams::load(a.cost_params);
  PerfLibrary lib;
  if (!a.perf_lib.empty() && std::ifstream(a.perf_lib).good()) lib = PerfLibrary::load(a.perf_lib);
  TensorGraph graph;
  try {
    graph = parse_graph(read_file(a.graph));
  } catch (const ParseError& e) {
    throw UsageError(a.graph + ": " + e.what());
  }
  const auto inputs = read_inputs(a.inputs, graph, a.options.seed);
  const CompileReport report = compile_graph(graph, a.options, lib, params);
  if (a.literal) stitchfuse_device::set_strategy(SFX_STRATEGY_LITERAL);
  const std::map<InstrId, TensorValue> values =
      a.host ? stitchfuse::run_compiled(report, graph, inputs) : stitchfuse_device::run_compiled(report, graph, inputs);
  for (const InstrId& o : graph.outputs()) {
    const TensorValue& v = values.at(o);
    std::cout << o << " shape=" << to_string(v.shape) << " checksum=" << checksum(v) << "\n";
    if (!a.dump) continue;
    const int64_t n = v.shape.element_count();
    for (int64_t i = 0; i < n; ++i)
      std::cout << (i ? " " : "  ")
                << (v.shape.etype == ElementType::F32 ? std::to_string(v.f32[i]) : std::to_string(v.i32[i]));
    std::cout << "\n";
  }
  if (a.compare) {
    const auto ref = interpret(graph, inputs);
    bool pass = true;
    for (const InstrId& o : graph.outputs())
      if (!close_enough(values.at(o), ref.at(o), 1e-5)) {
        std::cout << "MISMATCH " << o << "\n";
        pass = false;
      }
    std::cout << "reference check: " << (pass ? "PASS" : "FAIL") << "\n";
    if (!pass) return 2;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(parse_args(argc, argv));
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const ParseError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return 2;
  }
}
