// See stitchfuse_device.hpp.  Flattens the reference's TensorGraph /
// KernelProgram (ir.hpp:82-125, kernelgen.hpp:25-54) into the C-ABI
// descriptors of include/sfx.h and drives libsfx.so.
#include "stitchfuse_device.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <variant>

#include "sfx.h"
#include "stitchfuse/fixtures.hpp"
#include "stitchfuse/kernelgen.hpp"
#include "stitchfuse/schedule.hpp"
#include "stitchfuse/smem.hpp"
#include "stitchfuse/span.hpp"
#include "stitchfuse/tuning.hpp"
#include "json.hpp"

namespace stitchfuse_device {

using namespace stitchfuse;

namespace {

void check(sfx_status st) {
  if (st != SFX_OK) throw ExecError(std::string("device executor: ") + sfx_last_error());
}

sfx_ctx* context() {
  static sfx_ctx* ctx = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* d = std::getenv("SFX_DEVICE");
    check(sfx_ctx_create(d ? std::atoi(d) : 0, &ctx));
  });
  return ctx;
}

// Owns every array the descriptor points into.
struct Desc {
  std::vector<sfx_instr> instrs;
  std::vector<std::vector<double>> literals;
  std::vector<int32_t> outputs;
  std::vector<std::vector<int32_t>> members, roots;
  std::vector<std::vector<sfx_stmt>> stmts;
  std::vector<std::vector<sfx_member_plan>> plans;
  std::vector<sfx_program> programs;
  std::map<InstrId, int32_t> index;
  sfx_graph_desc desc{};

  Desc(const TensorGraph& g, const std::vector<const KernelProgram*>& progs) {
    const auto& ins = g.instructions();
    for (size_t i = 0; i < ins.size(); ++i) index[ins[i].id] = static_cast<int32_t>(i);
    instrs.resize(ins.size());
    literals.resize(ins.size());
    for (size_t i = 0; i < ins.size(); ++i) {
      const Instruction& in = ins[i];
      sfx_instr& s = instrs[i];
      std::memset(&s, 0, sizeof s);
      s.id = in.id.c_str();
      s.opcode = static_cast<int32_t>(in.opcode);  // same enumerator order (ir.hpp:41-52)
      s.kind = static_cast<int32_t>(in.kind);      // ir.hpp:54-73
      if (in.opcode == Opcode::LibraryCall)
        s.kind = in.callee == "matmul" ? SFX_CALLEE_MATMUL : in.callee == "opaque" ? SFX_CALLEE_OPAQUE : -1;
      s.dtype = in.shape.etype == ElementType::F32 ? SFX_F32 : SFX_I32;
      if (in.shape.rank() > SFX_MAX_RANK) throw ExecError("rank above SFX_MAX_RANK: " + in.id);
      s.rank = static_cast<int32_t>(in.shape.rank());
      for (int d = 0; d < s.rank; ++d) s.dims[d] = in.shape.dims[d];
      s.n_operands = static_cast<int32_t>(in.operands.size());
      for (int k = 0; k < s.n_operands && k < 3; ++k) s.operands[k] = index.at(in.operands[k]);
      for (size_t k = 0; k < in.permutation.size(); ++k) s.permutation[k] = in.permutation[k];
      s.n_dim_map = static_cast<int32_t>(in.broadcast_dim_map.size());
      for (size_t k = 0; k < in.broadcast_dim_map.size(); ++k) s.broadcast_dim_map[k] = in.broadcast_dim_map[k];
      s.n_reduce_dims = static_cast<int32_t>(in.reduce_dims.size());
      for (size_t k = 0; k < in.reduce_dims.size(); ++k) s.reduce_dims[k] = in.reduce_dims[k];
      s.reducer = static_cast<int32_t>(in.reducer);  // Sum, Max, Min (ir.hpp:75)
      s.scalar = in.scalar;
      literals[i] = in.literal;
      s.n_literal = static_cast<int64_t>(literals[i].size());
      s.literal = literals[i].empty() ? nullptr : literals[i].data();
    }
    for (const InstrId& o : g.outputs()) outputs.push_back(index.at(o));
    for (const KernelProgram* p : progs) {
      members.emplace_back();
      for (const InstrId& m : p->comp.members) members.back().push_back(index.at(m));
      roots.emplace_back();
      for (const InstrId& r : p->comp.roots) roots.back().push_back(index.at(r));
      stmts.emplace_back();
      for (const Statement& st : p->statements) {
        sfx_stmt t;
        std::memset(&t, 0, sizeof t);
        if (const auto* m = std::get_if<MaterializeStmt>(&st)) {
          t.kind = SFX_STMT_MATERIALIZE;
          t.instr = index.at(m->instr);
          t.split_dim = m->schedule.split_dim;
          t.sword = m->schedule.sword;
          t.sched_type = m->schedule.type == SchedType::Row ? SFX_SCHED_ROW : SFX_SCHED_COL;
          if (const auto* sh = std::get_if<SharedDest>(&m->dest)) {
            t.dest = SFX_DEST_SHARED;
            t.offset = sh->offset;
            t.bytes = sh->bytes;
          } else {
            t.dest = SFX_DEST_OUTPUT;
            t.root_index = std::get<OutputDest>(m->dest).root_index;
          }
        } else if (std::holds_alternative<BarrierStmt>(st)) {
          t.kind = SFX_STMT_BARRIER;
        } else {
          t.kind = SFX_STMT_INLINE;
          t.instr = index.at(std::get<InlineBindingStmt>(st).instr);
        }
        stmts.back().push_back(t);
      }
    }
    for (size_t k = 0; k < progs.size(); ++k) {
      const KernelProgram* p = progs[k];
      sfx_program sp;
      std::memset(&sp, 0, sizeof sp);
      sp.n_members = static_cast<int32_t>(members[k].size());
      sp.members = members[k].data();
      sp.n_roots = static_cast<int32_t>(roots[k].size());
      sp.roots = roots[k].data();
      sp.fusion_root = index.count(p->comp.fusion_root) ? index.at(p->comp.fusion_root) : -1;
      sp.blocks = p->plan.blocks;
      sp.block_threads = p->plan.block_threads;
      sp.arena_bytes = p->arena_bytes;
      sp.n_stmts = static_cast<int32_t>(stmts[k].size());
      sp.stmts = stmts[k].data();
      // the geometry reads use (exec.cpp:320-324), per member
      plans.emplace_back();
      for (const InstrId& m : p->comp.members) {
        sfx_member_plan mp{};
        auto off = p->arena_offsets.find(m);
        mp.arena_offset = off == p->arena_offsets.end() ? -1 : off->second;
        auto sc = p->plan.per_instruction.find(m);
        if (sc != p->plan.per_instruction.end()) {
          mp.split_dim = sc->second.split_dim;
          mp.sword = sc->second.sword;
          mp.sched_type = sc->second.type == SchedType::Row ? SFX_SCHED_ROW : SFX_SCHED_COL;
        } else {
          mp.sword = 1;
        }
        plans.back().push_back(mp);
      }
      sp.member_plans = plans.back().data();
      programs.push_back(sp);
    }
    desc.n_instrs = static_cast<int32_t>(instrs.size());
    desc.instrs = instrs.data();
    desc.n_outputs = static_cast<int32_t>(outputs.size());
    desc.outputs = outputs.data();
    desc.n_programs = static_cast<int32_t>(programs.size());
    desc.programs = programs.data();
  }

  // Plan signature: every byte the lowering reads (the descriptors with their
  // pointers replaced by the pointed-to contents) plus the options.  Equal
  // signatures compile to the same kernels, so the compiled object is reused.
  std::string signature(const sfx_compile_opts& o) const {
    std::string k;
    auto put = [&](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
    put(&o, sizeof o);
    for (size_t i = 0; i < instrs.size(); ++i) {
      sfx_instr c = instrs[i];  // memset-initialised: padding is zero
      c.id = nullptr;
      c.literal = nullptr;
      put(&c, sizeof c);
      k.append(instrs[i].id).push_back('\0');
      put(literals[i].data(), literals[i].size() * sizeof(double));
    }
    put(outputs.data(), outputs.size() * sizeof(int32_t));
    for (size_t p = 0; p < programs.size(); ++p) {
      sfx_program sp = programs[p];
      sp.members = sp.roots = nullptr;
      sp.stmts = nullptr;
      sp.member_plans = nullptr;
      put(&sp, sizeof sp);
      put(members[p].data(), members[p].size() * sizeof(int32_t));
      put(roots[p].data(), roots[p].size() * sizeof(int32_t));
      put(stmts[p].data(), stmts[p].size() * sizeof(sfx_stmt));
      put(plans[p].data(), plans[p].size() * sizeof(sfx_member_plan));
    }
    return k;
  }
};

// Compiled kernels / modules by plan signature, least recently used evicted
// beyond SFX_BINDING_CACHE entries (default 8; a cached module keeps its device
// intermediates and host-path staging buffers; 0 = compile every call).
// Entries are shared_ptrs: an evicted object lives until its last user returns.
template <typename T>
class Cache {
 public:
  explicit Cache(sfx_status (*destroy)(T*)) : destroy_(destroy) {
    const char* e = std::getenv("SFX_BINDING_CACHE");
    cap_ = e ? std::max(0, std::atoi(e)) : 8;
  }
  std::shared_ptr<T> get(const std::string& key, const std::function<T*()>& make) {
    std::lock_guard<std::mutex> lock(mu_);
    auto it = map_.find(key);
    if (it != map_.end()) {
      it->second.second = ++tick_;
      return it->second.first;
    }
    auto destroy = destroy_;
    std::shared_ptr<T> obj(make(), [destroy](T* p) { destroy(p); });
    ++compiles_;
    if (cap_ == 0) return obj;
    if (map_.size() >= static_cast<size_t>(cap_)) {
      auto lru = map_.begin();
      for (auto j = map_.begin(); j != map_.end(); ++j)
        if (j->second.second < lru->second.second) lru = j;
      map_.erase(lru);
    }
    map_.emplace(key, std::make_pair(obj, ++tick_));
    return obj;
  }
  long long compiles() {
    std::lock_guard<std::mutex> lock(mu_);
    return compiles_;
  }

 private:
  sfx_status (*destroy_)(T*);
  int cap_ = 8;
  unsigned long long tick_ = 0;
  long long compiles_ = 0;
  std::map<std::string, std::pair<std::shared_ptr<T>, unsigned long long>> map_;
  std::mutex mu_;
};

// Never destroyed (process exit reclaims device memory; destroying modules
// after the CUDA context is gone would fail).
Cache<sfx_kernel>& kernel_cache() {
  static auto* c = new Cache<sfx_kernel>(&sfx_kernel_destroy);
  return *c;
}
Cache<sfx_graph>& graph_cache() {
  static auto* c = new Cache<sfx_graph>(&sfx_graph_destroy);
  return *c;
}

const void* host_data(const TensorValue& v) {
  return v.shape.etype == ElementType::F32 ? static_cast<const void*>(v.f32.data())
                                           : static_cast<const void*>(v.i32.data());
}
void* host_data(TensorValue& v) {
  return v.shape.etype == ElementType::F32 ? static_cast<void*>(v.f32.data()) : static_cast<void*>(v.i32.data());
}

sfx_compile_opts g_opts{};

}  // namespace

long long launches() { return sfx_launch_count(context()); }
long long compiles() { return kernel_cache().compiles() + graph_cache().compiles(); }
void set_strategy(int sfx_strategy) { g_opts.strategy = sfx_strategy; }
void set_debug_checks(int level) { g_opts.debug_checks = level; }

std::vector<TensorValue> run_program(const KernelProgram& program, const TensorGraph& graph,
                                     const std::map<InstrId, TensorValue>& externals) {
  sfx_ctx* ctx = context();
  Desc d(graph, {&program});
  std::shared_ptr<sfx_kernel> kp = kernel_cache().get(d.signature(g_opts), [&] {
    sfx_kernel* nk = nullptr;
    check(sfx_program_compile(ctx, &d.desc, 0, &g_opts, &nk));
    return nk;
  });
  sfx_kernel* k = kp.get();
  sfx_kernel_info info;
  check(sfx_kernel_get_info(k, &info));
  std::vector<int32_t> slots(info.n_inputs);
  check(sfx_kernel_input_instrs(k, slots.data(), info.n_inputs));
  std::vector<uint64_t> in, out;
  auto free_all = [&] {
    for (uint64_t p : in) sfx_free(ctx, p);
    for (uint64_t p : out) sfx_free(ctx, p);
  };
  try {
    for (int32_t s : slots) {
      const InstrId& id = graph.instructions()[s].id;
      auto it = externals.find(id);
      if (it == externals.end()) throw ExecError("missing external value " + id);
      uint64_t p = 0;
      uint64_t bytes = static_cast<uint64_t>(it->second.shape.byte_size());
      check(sfx_alloc(ctx, bytes, &p));
      in.push_back(p);
      check(sfx_memcpy_h2d(ctx, p, host_data(it->second), bytes, nullptr));
    }
    std::vector<TensorValue> res;
    for (const InstrId& r : program.comp.roots) {
      res.push_back(TensorValue::zeros(graph.at(r).shape));
      uint64_t p = 0;
      check(sfx_alloc(ctx, static_cast<uint64_t>(graph.at(r).shape.byte_size()), &p));
      out.push_back(p);
    }
    check(sfx_program_launch(k, in.data(), static_cast<int32_t>(in.size()), out.data(),
                             static_cast<int32_t>(out.size()), nullptr));
    for (size_t i = 0; i < res.size(); ++i)
      check(sfx_memcpy_d2h(ctx, host_data(res[i]), out[i], static_cast<uint64_t>(res[i].shape.byte_size()), nullptr));
    check(sfx_stream_sync(ctx, nullptr));
    free_all();
    return res;
  } catch (...) {
    free_all();
    throw;
  }
}

std::map<InstrId, TensorValue> run_compiled(const CompileReport& report, const TensorGraph& graph,
                                            const std::map<InstrId, TensorValue>& inputs) {
  sfx_ctx* ctx = context();
  std::vector<const KernelProgram*> progs;
  for (const CompiledKernel& k : report.kernels) progs.push_back(&k.program);
  Desc d(graph, progs);
  std::shared_ptr<sfx_graph> gp = graph_cache().get(d.signature(g_opts), [&] {
    sfx_graph* ng = nullptr;
    check(sfx_graph_compile(ctx, &d.desc, &g_opts, &ng));
    return ng;
  });
  sfx_graph* g = gp.get();
  int32_t n = 0;
  std::vector<int32_t> params(graph.instructions().size());
  check(sfx_graph_param_instrs(g, params.data(), static_cast<int32_t>(params.size()), &n));
  std::vector<const void*> pin;
  for (int32_t i = 0; i < n; ++i) {
    const InstrId& id = graph.instructions()[params[i]].id;
    auto it = inputs.find(id);
    if (it == inputs.end()) throw ExecError("missing input for parameter " + id);
    if (it->second.shape != graph.at(id).shape) throw ExecError("input shape mismatch for " + id);
    pin.push_back(host_data(it->second));
  }
  std::map<InstrId, TensorValue> values;
  std::vector<void*> pout;
  for (const InstrId& o : graph.outputs()) values[o] = TensorValue::zeros(graph.at(o).shape);
  for (const InstrId& o : graph.outputs()) pout.push_back(host_data(values[o]));
  check(sfx_graph_run_host(g, pin.data(), n, pout.data(), static_cast<int32_t>(pout.size()), nullptr));
  // The rest of the reference's map (pipeline.cpp:104-118): parameters and
  // constants from the host, every other group root and unfused instruction
  // read back from HBM (intermediates stay device-resident during the run).
  std::set<InstrId> members;
  for (const CompiledKernel& k : report.kernels) members.insert(k.comp.members.begin(), k.comp.members.end());
  std::set<InstrId> roots;
  for (const CompiledKernel& k : report.kernels) roots.insert(k.comp.roots.begin(), k.comp.roots.end());
  for (const Instruction& ins : graph.instructions()) {
    if (values.count(ins.id)) continue;
    if (ins.opcode == Opcode::Parameter) {
      values[ins.id] = inputs.at(ins.id);
    } else if (ins.opcode == Opcode::Constant) {
      values[ins.id] = constant_value(ins);
    } else if (roots.count(ins.id) || !members.count(ins.id)) {
      TensorValue v = TensorValue::zeros(ins.shape);
      check(sfx_graph_fetch(g, d.index.at(ins.id), host_data(v), static_cast<uint64_t>(ins.shape.byte_size()),
                            nullptr));
      values[ins.id] = std::move(v);
    }
  }
  return values;
}

// ---- measured perf library ---------------------------------------------------

namespace {

// A graph holding one instruction of `g` with its operands as parameters.
TensorGraph single_instruction_graph(const TensorGraph& g, const Instruction& ins) {
  nlohmann::json doc = nlohmann::json::parse(serialize_graph(g));
  nlohmann::json one;
  for (const auto& j : doc["instructions"])
    if (j["id"] == ins.id) one = j;
  nlohmann::json out = {{"instructions", nlohmann::json::array()}, {"outputs", {ins.id}}};
  std::vector<std::string> ops;
  for (size_t k = 0; k < ins.operands.size(); ++k) {
    const Shape& sh = g.at(ins.operands[k]).shape;
    const std::string pid = "in" + std::to_string(k);
    nlohmann::json p = {{"id", pid}, {"op", "parameter"}, {"shape", sh.dims}};
    if (sh.etype == ElementType::I32) p["dtype"] = "i32";
    out["instructions"].push_back(p);
    ops.push_back(pid);
  }
  one["operands"] = ops;
  out["instructions"].push_back(one);
  return parse_graph(out.dump());
}

}  // namespace

MeasureStats measure_misses(const TensorGraph& graph, const PipelineOptions& options, PerfLibrary& lib,
                            const CostModelParams& params, int reps, int max_keys) {
  MeasureStats st;
  sfx_ctx* ctx = context();
  sfx_compile_opts lit{};
  lit.strategy = SFX_STRATEGY_LITERAL;
  // Measured costs move the planner's tuned schedules, and a new schedule is a
  // new key: re-plan with what was measured and measure the new misses, until a
  // plan misses nothing new (every miss is measured once, as the paper's
  // on-miss path does one key at a time).
  std::set<PerfKey> tried;
  for (int round = 0; round < 16; ++round) {
    PerfLibrary probe = lib;
    compile_graph(graph, options, probe, params);  // misses become synthetic entries
    bool fresh = false;
    for (const auto& [key, entry] : probe.entries()) {
      const PerfEntry* have = lib.find(key);
      if (!entry.synthetic || (have && !have->synthetic)) continue;
      if (!tried.insert(key).second) continue;
      fresh = true;
      ++st.keys_missed;
      if (max_keys >= 0 && st.keys_measured >= max_keys) continue;
      const Instruction* ins = nullptr;
      for (const Instruction& i : graph.instructions())
        if (opcode_name(i) == key.opcode && i.shape.dims == key.shape) {
          ins = &i;
          break;
        }
      if (!ins) continue;
      try {
        TensorGraph g1 = single_instruction_graph(graph, *ins);
        PipelineOptions o1 = options;
        o1.fuse_dot = true;  // a lone BatchMatMul key is measured as its own group
        FusionPlan fp = fuse_module(g1, o1);
        const FusedComputation* comp = nullptr;
        for (const FusedComputation& c : fp.computations)
          if (c.members.count(ins->id)) comp = &c;
        if (!comp) continue;
        Schedule sched;
        sched.split_dim = key.split_dim;
        sched.sword = key.sword;
        sched.type = key.sched_type;
        ResolveResult r = resolve_schedule(*comp, g1, {{ins->id, sched}}, o1);
        if (!r.ok()) continue;
        SchedulePlan plan = *r.plan;
        plan.block_threads = key.block_threads;
        SpanMap sm = compute_span(g1);
        SmemResult smem = plan_shared_memory(*comp, g1, sm, plan, o1);
        if (!std::holds_alternative<SharedMemPlan>(smem)) continue;
        KernelProgram prog = emit_program(*comp, g1, sm, plan, std::get<SharedMemPlan>(smem), o1);
        Desc d(g1, {&prog});
        double us = 0;
        check(sfx_program_time(ctx, &d.desc, 0, &lit, reps, &us, nullptr));
        PerfEntry e;
        e.cost_us = us;
        e.synthetic = false;
        lib.insert(key, e);
        ++st.keys_measured;
      } catch (const std::exception& e) {
        st.notes.push_back(key.opcode + ": " + e.what());
      }
    }
    if (!fresh) break;
  }
  return st;
}

MeasureStats tune_templates(const CompileReport& report, const TensorGraph& graph, int reps) {
  MeasureStats st;
  sfx_ctx* ctx = context();
  std::vector<const KernelProgram*> progs;
  for (const CompiledKernel& k : report.kernels) progs.push_back(&k.program);
  Desc d(graph, progs);
  for (size_t i = 0; i < progs.size(); ++i) {
    const int32_t pi = static_cast<int32_t>(i);
    sfx_compile_opts dflt{};
    char sig[512];
    check(sfx_program_signature(&d.desc, pi, &dflt, sig, sizeof sig));
    if (sfx_template_param_has(sig)) continue;  // hit
    std::string strategy(256, '\0');
    check(sfx_program_codegen(&d.desc, pi, &dflt, nullptr, 0, nullptr, 0, strategy.data(), strategy.size()));
    strategy = strategy.substr(0, strategy.find(' '));
    std::vector<sfx_compile_opts> cands;
    auto cand = [&](int rows, int tpr, int items, int ctas) {
      sfx_compile_opts o{};
      o.rows_per_cta = rows;
      o.threads_per_row = tpr;
      o.items_per_thread = items;
      o.pipe_ctas_per_sm = ctas;
      cands.push_back(o);
    };
    if (strategy == "map") {
      for (int u : {1, 2, 4, 8}) cand(0, 0, u, 0);
    } else if (strategy == "row") {
      for (int t : {32, 64, 128, 256}) cand(0, t, 0, 0);
      for (int r : {1, 2, 4}) cand(r, 0, 0, 0);
      for (int t : {64, 128})
        for (int r : {1, 4}) cand(r, t, 0, 0);
    } else if (strategy == "col") {
      cand(0, 0, 24, 1), cand(0, 0, 32, 1), cand(0, 0, 8, 2), cand(0, 0, 12, 3);
    } else {
      continue;  // literal / colbc / dot: no template knobs
    }
    double t0 = 0, c0 = 0;
    check(sfx_program_time(ctx, &d.desc, pi, &dflt, reps, &t0, &c0));
    ++st.groups_tuned;
    double best = t0;
    const sfx_compile_opts* win = nullptr;
    for (const sfx_compile_opts& o : cands) {
      double t = 0, c = 0;
      if (sfx_program_time(ctx, &d.desc, pi, &o, reps, &t, &c) != SFX_OK) continue;  // knob not applicable
      if (!(std::abs(c - c0) <= 1e-4 * std::max(1.0, std::abs(c0)))) continue;   // must compute the same
      if (t < 0.98 * t0 && t < best) best = t, win = &o;
    }
    const std::string root = progs[i]->comp.fusion_root;
    if (win) {
      check(sfx_template_param_put(sig, win->rows_per_cta, win->threads_per_row, win->items_per_thread,
                                   win->pipe_ctas_per_sm, best, t0, ("measured on miss: " + root).c_str()));
      ++st.groups_changed;
      st.notes.push_back(root + ": " + sig + " " + std::to_string(t0) + " -> " + std::to_string(best) + " us");
    } else {
      check(sfx_template_param_put(sig, 0, 0, 0, 0, t0, t0, ("measured on miss, defaults kept: " + root).c_str()));
      st.notes.push_back(root + ": " + sig + " defaults kept (" + std::to_string(t0) + " us)");
    }
  }
  return st;
}

std::string template_params_text() {
  uint64_t need = 0;
  check(sfx_template_params_text(nullptr, 0, &need));
  std::string t(need, '\0');
  check(sfx_template_params_text(t.data(), t.size(), &need));
  t.resize(need ? need - 1 : 0);
  return t;
}

}  // namespace stitchfuse_device
