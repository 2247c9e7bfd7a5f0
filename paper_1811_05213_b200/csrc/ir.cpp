// Descriptor -> internal graph, with the reference's shape validation
// (reference proj/src/ir.cpp:215-323) and KernelProgram structure checks
// (reference proj/src/kernelgen.cpp:75-104).
#include "ir.hpp"

#include <algorithm>
#include <map>

namespace sfx {

const char* ew_name(int kind) {
  static const char* names[] = {"add", "sub", "mul",   "max",  "min", "neg",  "compare", "select",
                                "scale", "exp", "log", "div", "pow", "tanh", "sqrt", "rsqrt"};
  if (kind < 0 || kind > SFX_EW_RSQRT) return "?";
  return names[kind];
}

// reference ir.cpp:47-62
int ew_arity(int kind) {
  switch (kind) {
    case SFX_EW_NEG: case SFX_EW_SCALE: case SFX_EW_EXP: case SFX_EW_LOG: case SFX_EW_TANH:
    case SFX_EW_SQRT: case SFX_EW_RSQRT:
      return 1;
    case SFX_EW_SELECT:
      return 3;
    default:
      return 2;
  }
}

namespace {

[[noreturn]] void bad(const std::string& what) { throw Error(SFX_ERR_INVALID, what); }

bool expensive(int kind) { return kind >= SFX_EW_EXP; }

void validate_node(const Graph& g, const Node& n) {
  auto in = [&](size_t i) -> const Node& { return g.nodes[n.operands[i]]; };
  for (int64_t d : n.dims)
    if (d < 1) bad("instruction " + n.id + ": dimension extents must be >= 1");
  switch (n.op) {
    case SFX_OP_PARAMETER:
    case SFX_OP_CONSTANT:
      if (!n.operands.empty()) bad("instruction " + n.id + ": takes no operands");
      if (n.op == SFX_OP_CONSTANT && n.literal.size() != 1 &&
          static_cast<int64_t>(n.literal.size()) != n.numel())
        bad("instruction " + n.id + ": constant literal size mismatch");
      break;
    case SFX_OP_ELEMENTWISE:
      if (n.kind < 0 || n.kind > SFX_EW_RSQRT) bad("instruction " + n.id + ": bad elementwise kind");
      if (static_cast<int>(n.operands.size()) != ew_arity(n.kind))
        bad("instruction " + n.id + ": wrong operand count");
      for (size_t i = 0; i < n.operands.size(); ++i)
        if (in(i).dims != n.dims || in(i).dtype != n.dtype)
          bad("instruction " + n.id + ": operand shape mismatch (no implicit broadcast)");
      if (n.dtype == SFX_I32 && expensive(n.kind)) bad("instruction " + n.id + ": requires f32");
      break;
    case SFX_OP_RESHAPE:
    case SFX_OP_BITCAST:
      if (n.operands.size() != 1) bad("instruction " + n.id + ": expects 1 operand");
      if (in(0).numel() != n.numel()) bad("instruction " + n.id + ": element count mismatch");
      if (n.op == SFX_OP_RESHAPE && in(0).dtype != n.dtype)
        bad("instruction " + n.id + ": element type mismatch");
      break;
    case SFX_OP_TRANSPOSE: {
      if (n.operands.size() != 1) bad("instruction " + n.id + ": expects 1 operand");
      const Node& s = in(0);
      if (static_cast<int>(n.perm.size()) != n.rank() || s.rank() != n.rank())
        bad("instruction " + n.id + ": permutation rank mismatch");
      std::vector<bool> seen(n.perm.size(), false);
      for (int64_t p : n.perm) {
        if (p < 0 || p >= n.rank() || seen[p]) bad("instruction " + n.id + ": permutation not bijective");
        seen[p] = true;
      }
      for (int i = 0; i < n.rank(); ++i)
        if (n.dims[i] != s.dims[n.perm[i]]) bad("instruction " + n.id + ": permuted shape mismatch");
      break;
    }
    case SFX_OP_BROADCAST: {
      if (n.operands.size() != 1) bad("instruction " + n.id + ": expects 1 operand");
      const Node& s = in(0);
      if (static_cast<int>(n.dim_map.size()) != s.rank()) bad("instruction " + n.id + ": dim_map size");
      int64_t prev = -1;
      for (size_t i = 0; i < n.dim_map.size(); ++i) {
        int64_t d = n.dim_map[i];
        if (d <= prev || d >= n.rank()) bad("instruction " + n.id + ": dim_map not increasing");
        if (n.dims[d] != s.dims[i]) bad("instruction " + n.id + ": mapped extent mismatch");
        prev = d;
      }
      break;
    }
    case SFX_OP_REDUCE: {
      if (n.operands.size() != 1) bad("instruction " + n.id + ": expects 1 operand");
      const Node& s = in(0);
      std::set<int64_t> rd(n.reduce_dims.begin(), n.reduce_dims.end());
      if (rd.size() != n.reduce_dims.size()) bad("instruction " + n.id + ": reduce_dims not distinct");
      std::vector<int64_t> expect;
      for (int i = 0; i < s.rank(); ++i)
        if (!rd.count(i)) expect.push_back(s.dims[i]);
      for (int64_t d : rd)
        if (d < 0 || d >= s.rank()) bad("instruction " + n.id + ": reduce dim out of range");
      if (expect != n.dims) bad("instruction " + n.id + ": reduce output shape mismatch");
      if (n.reducer < 0 || n.reducer > SFX_REDUCE_MIN) bad("instruction " + n.id + ": bad reducer");
      break;
    }
    case SFX_OP_LIBRARY_CALL:
      if (n.kind == SFX_CALLEE_OPAQUE) break;  // a barrier only (ir.cpp:316-317)
      if (n.kind != SFX_CALLEE_MATMUL) bad("instruction " + n.id + ": unknown library callee");
      [[fallthrough]];
    case SFX_OP_BATCH_MATMUL: {
      // reference ir.cpp:288-315: [..., M, K] x [..., K, N] -> [..., M, N]
      const int min_rank = n.op == SFX_OP_BATCH_MATMUL ? 3 : 2;
      if (n.operands.size() != 2) bad("instruction " + n.id + ": matmul expects 2 operands");
      const Node& a = in(0);
      const Node& b = in(1);
      const int r = a.rank();
      if (r < min_rank || b.rank() != r || n.rank() != r)
        bad("instruction " + n.id + ": operand ranks must be equal and >= " + std::to_string(min_rank));
      for (int i = 0; i < r - 2; ++i)
        if (a.dims[i] != b.dims[i] || a.dims[i] != n.dims[i]) bad("instruction " + n.id + ": batch dims mismatch");
      if (a.dims[r - 1] != b.dims[r - 2]) bad("instruction " + n.id + ": contraction extents mismatch");
      if (n.dims[r - 2] != a.dims[r - 2] || n.dims[r - 1] != b.dims[r - 1])
        bad("instruction " + n.id + ": output dims mismatch");
      if (a.dtype != n.dtype || b.dtype != n.dtype) bad("instruction " + n.id + ": element type mismatch");
      break;
    }
    default:
      bad("instruction " + n.id + ": unknown opcode");
  }
}

}  // namespace

Graph graph_from_desc(const sfx_graph_desc* d) {
  if (!d) bad("null graph descriptor");
  if (d->n_instrs < 0 || (d->n_instrs > 0 && !d->instrs)) bad("bad instruction array");
  Graph g;
  g.nodes.resize(d->n_instrs);
  std::map<std::string, int> by_id;
  for (int i = 0; i < d->n_instrs; ++i) {
    const sfx_instr& s = d->instrs[i];
    Node& n = g.nodes[i];
    n.id = s.id ? s.id : ("#" + std::to_string(i));
    if (!by_id.emplace(n.id, i).second) bad("duplicate instruction id " + n.id);
    n.op = s.opcode;
    n.kind = s.kind;
    n.dtype = s.dtype;
    if (s.dtype != SFX_F32 && s.dtype != SFX_I32) bad("instruction " + n.id + ": bad dtype");
    if (s.rank < 0 || s.rank > SFX_MAX_RANK) bad("instruction " + n.id + ": bad rank");
    n.dims.assign(s.dims, s.dims + s.rank);
    if (s.n_operands < 0 || s.n_operands > 3) bad("instruction " + n.id + ": bad operand count");
    for (int k = 0; k < s.n_operands; ++k) {
      if (s.operands[k] < 0 || s.operands[k] >= d->n_instrs)
        bad("instruction " + n.id + ": operand index out of range");
      n.operands.push_back(s.operands[k]);
    }
    if (n.op == SFX_OP_TRANSPOSE) n.perm.assign(s.permutation, s.permutation + s.rank);
    if (s.n_dim_map < 0 || s.n_dim_map > SFX_MAX_RANK) bad("instruction " + n.id + ": bad dim map");
    n.dim_map.assign(s.broadcast_dim_map, s.broadcast_dim_map + s.n_dim_map);
    if (s.n_reduce_dims < 0 || s.n_reduce_dims > SFX_MAX_RANK) bad("instruction " + n.id + ": bad reduce dims");
    n.reduce_dims.assign(s.reduce_dims, s.reduce_dims + s.n_reduce_dims);
    n.reducer = s.reducer;
    n.scalar = s.scalar;
    if (s.n_literal > 0) {
      if (!s.literal) bad("instruction " + n.id + ": null literal");
      n.literal.assign(s.literal, s.literal + s.n_literal);
    }
  }
  g.users.resize(g.nodes.size());
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    std::set<int> seen;
    for (int op : g.nodes[i].operands)
      if (seen.insert(op).second) g.users[op].push_back(static_cast<int>(i));
  }
  for (const Node& n : g.nodes) validate_node(g, n);
  for (int k = 0; k < d->n_outputs; ++k) {
    int o = d->outputs[k];
    if (o < 0 || o >= d->n_instrs) bad("output index out of range");
    g.outputs.push_back(o);
  }

  auto id_less = [&](int a, int b) { return g.nodes[a].id < g.nodes[b].id; };
  for (int p = 0; p < d->n_programs; ++p) {
    const sfx_program& sp = d->programs[p];
    Program pr;
    for (int k = 0; k < sp.n_members; ++k) {
      int m = sp.members[k];
      if (m < 0 || m >= d->n_instrs) bad("program member out of range");
      pr.member_set.insert(m);
    }
    pr.members.assign(pr.member_set.begin(), pr.member_set.end());
    std::sort(pr.members.begin(), pr.members.end(), id_less);
    for (int k = 0; k < sp.n_roots; ++k) {
      int r = sp.roots[k];
      if (!pr.member_set.count(r)) bad("program root is not a member");
      pr.roots.push_back(r);
    }
    pr.fusion_root = sp.fusion_root;
    pr.blocks = sp.blocks;
    pr.block_threads = sp.block_threads;
    pr.arena_bytes = sp.arena_bytes;
    if (pr.blocks < 1) bad("program blocks must be >= 1");
    for (int k = 0; k < sp.n_stmts; ++k) {
      const sfx_stmt& s = sp.stmts[k];
      Stmt st;
      st.kind = s.kind;
      st.instr = s.instr;
      st.split_dim = s.split_dim;
      st.sword = s.sword;
      st.sched = s.sched_type;
      st.dest = s.dest;
      st.offset = s.offset;
      st.bytes = s.bytes;
      st.root_index = s.root_index;
      if (st.kind != SFX_STMT_BARRIER) {
        if (!pr.member_set.count(st.instr)) bad("statement instruction is not a member");
      }
      pr.stmts.push_back(st);
    }
    std::set<int> ext;
    for (int m : pr.members) {
      const Node& n = g.nodes[m];
      if (n.op == SFX_OP_PARAMETER || n.op == SFX_OP_CONSTANT)
        bad("program member " + n.id + " is a parameter/constant");
      for (int op : n.operands)
        if (!pr.member_set.count(op)) ext.insert(op);
    }
    pr.externals.assign(ext.begin(), ext.end());
    std::sort(pr.externals.begin(), pr.externals.end(), id_less);
    for (int e : pr.externals)
      if (!g.nodes[e].is_splat()) pr.inputs.push_back(e);
    // kernelgen.cpp:75-104 — producer-before-consumer, arena bounds, roots once
    std::set<int> available;
    std::set<int> roots_written;
    for (const Stmt& st : pr.stmts) {
      if (st.kind == SFX_STMT_BARRIER) continue;
      for (int op : g.nodes[st.instr].operands)
        if (pr.member_set.count(op) && !available.count(op))
          bad("operand " + g.nodes[op].id + " of " + g.nodes[st.instr].id + " not yet available");
      if (st.kind == SFX_STMT_MATERIALIZE) {
        if (st.dest == SFX_DEST_SHARED) {
          if (st.offset < 0 || st.offset + st.bytes > pr.arena_bytes)
            bad("arena overflow for " + g.nodes[st.instr].id);
        } else {
          if (st.root_index < 0 || st.root_index >= static_cast<int>(pr.roots.size()) ||
              pr.roots[st.root_index] != st.instr)
            bad("root index mismatch for " + g.nodes[st.instr].id);
          if (!roots_written.insert(st.root_index).second)
            bad("root written twice: " + g.nodes[st.instr].id);
        }
      }
      available.insert(st.instr);
    }
    if (roots_written.size() != pr.roots.size()) bad("not all roots written");
    for (const Stmt& st : pr.stmts)
      if (st.kind == SFX_STMT_MATERIALIZE) {
        Program::ReadPlan rp;
        rp.offset = st.dest == SFX_DEST_SHARED ? st.offset : -1;
        rp.split_dim = st.split_dim;
        rp.sword = st.sword;
        rp.sched = st.sched;
        pr.reads[st.instr] = rp;
      }
    if (sp.member_plans)
      for (int k = 0; k < sp.n_members; ++k) {
        const sfx_member_plan& mp = sp.member_plans[k];
        Program::ReadPlan rp;
        rp.offset = mp.arena_offset;
        rp.split_dim = mp.split_dim;
        rp.sword = mp.sword;
        rp.sched = mp.sched_type;
        if (pr.reads.count(sp.members[k])) pr.reads[sp.members[k]] = rp;
      }
    check_executor_geometry(g, pr);
    g.programs.push_back(std::move(pr));
  }
  return g;
}

// The reference executor's run-time self-checks (exec.cpp:320-327, 399, 410)
// depend only on the program's geometry, never on data, so they are decided
// here, once, with the reference's messages and in the order its block loop
// would hit them: reads of arena members in block 0 (containment, then stale
// owner bytes), then a root overlap (a later block repeating a box), then
// incomplete coverage after the last block.
void check_executor_geometry(const Graph& g, const Program& pr) {
  auto blocks_of = [&](const Node& n, int64_t sd, int64_t sword, int sched) {
    int64_t prod = 1;
    if (n.rank() == 0) return int64_t{1};
    if (sched == SFX_SCHED_ROW)
      for (int64_t i = 0; i < sd; ++i) prod *= n.dims[i];
    else
      for (int64_t i = sd + 1; i < n.rank(); ++i) prod *= n.dims[i];
    return sword * prod;
  };
  auto box_elems = [&](const Node& n, int64_t sd, int64_t sword, int sched) {
    if (n.rank() == 0) return int64_t{1};
    int64_t e = n.dims[sd] / sword;
    if (sched == SFX_SCHED_ROW)
      for (int64_t i = sd + 1; i < n.rank(); ++i) e *= n.dims[i];
    else
      for (int64_t i = 0; i < sd; ++i) e *= n.dims[i];
    return e;
  };
  for (const Stmt& st : pr.stmts) {
    if (st.kind != SFX_STMT_MATERIALIZE) continue;
    const Node& n = g.nodes[st.instr];
    if (n.rank() > 0 && (st.split_dim < 0 || st.split_dim >= n.rank() || st.sword < 1))
      throw Error(SFX_ERR_INVALID, "invalid schedule for " + n.id);
  }
  std::vector<int> owner(static_cast<size_t>(std::max<int64_t>(pr.arena_bytes, 0)), -1);
  std::set<int> ready;
  std::map<int, const Stmt*> written;  // the (shared) statement that materialised a ready member
  std::string overlap, coverage;
  for (const Stmt& st : pr.stmts) {
    if (st.kind != SFX_STMT_MATERIALIZE) continue;
    // ready members this statement's evaluation reads (eval_element recursion)
    std::set<int> seen, reads;
    std::vector<int> stack{st.instr};
    while (!stack.empty()) {
      int m = stack.back();
      stack.pop_back();
      if (!pr.is_member(m) || !seen.insert(m).second) continue;
      if (ready.count(m)) {
        reads.insert(m);
        continue;
      }
      for (int op : g.nodes[m].operands) stack.push_back(op);
    }
    for (int r : reads) {
      const Node& rn = g.nodes[r];
      const Program::ReadPlan& rp = pr.reads.at(r);
      const Stmt& wp = *written.at(r);
      if (rp.split_dim != wp.split_dim || rp.sword != wp.sword || rp.sched != wp.sched)
        throw Error(SFX_ERR_EXEC, "chunk containment violation reading " + rn.id);
      const int64_t len = box_elems(rn, rp.split_dim, rp.sword, rp.sched) * 4;
      if (rp.offset < 0 || rp.offset + len > static_cast<int64_t>(owner.size()))
        throw Error(SFX_ERR_EXEC, "stale arena read of " + rn.id);
      for (int64_t b = rp.offset; b < rp.offset + len; ++b)
        if (owner[b] != r) throw Error(SFX_ERR_EXEC, "stale arena read of " + rn.id);
    }
    const Node& n = g.nodes[st.instr];
    if (st.dest == SFX_DEST_SHARED) {
      // a shared write drops ready members whose (read) buffers it overlaps
      const int64_t bytes = box_elems(n, st.split_dim, st.sword, st.sched) * 4;
      for (auto it = ready.begin(); it != ready.end();) {
        const Program::ReadPlan& rp = pr.reads.at(*it);
        const int64_t len = g.nodes[*it].numel() / pr.blocks * 4;
        if (*it != st.instr && rp.offset < st.offset + bytes && st.offset < rp.offset + len)
          it = ready.erase(it);
        else
          ++it;
      }
      if (st.offset + bytes > static_cast<int64_t>(owner.size()))
        throw Error(SFX_ERR_INVALID, "arena overflow for " + n.id);
      for (int64_t b = st.offset; b < st.offset + bytes; ++b) owner[b] = st.instr;
      ready.insert(st.instr);
      written[st.instr] = &st;
    } else {
      const int64_t nb = blocks_of(n, st.split_dim, st.sword, st.sched);
      if (nb < pr.blocks && overlap.empty()) overlap = "overlapping write to root " + n.id;
      if ((nb > pr.blocks || (n.rank() > 0 && n.dims[st.split_dim] % st.sword)) && coverage.empty())
        coverage = "incomplete coverage of root " + n.id;
    }
  }
  if (!overlap.empty()) throw Error(SFX_ERR_EXEC, overlap);
  if (!coverage.empty()) throw Error(SFX_ERR_EXEC, coverage);
}

}  // namespace sfx
