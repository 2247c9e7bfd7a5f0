// Literal tier: the reference KernelProgram executed as written.
#include "lower_impl.hpp"

namespace sfx {
namespace lw {

// ---- LITERAL --------------------------------------------------------------------

// chunk_box geometry (reference schedule.cpp:52-76) for a materialised member
struct Box {
  std::vector<std::string> lo;
  std::vector<int64_t> len;
};

Box chunk_box(Emitter& em, const Node& n, const Stmt& s, const std::string& blk) {
  Box b;
  const int rank = n.rank();
  b.lo.assign(rank, "0");
  b.len = n.dims;
  if (rank == 0) return b;
  const int64_t sd = s.split_dim;
  const int64_t slice_len = n.dims[sd] / s.sword;
  std::string slice = em.ivar(Emitter::imod(blk, s.sword));
  std::string fixed = em.ivar(Emitter::idiv(blk, s.sword));
  b.lo[sd] = em.ivar(Emitter::imul(slice, slice_len));
  b.len[sd] = slice_len;
  if (s.sched == SFX_SCHED_ROW) {
    for (int64_t i = sd - 1; i >= 0; --i) {
      b.lo[i] = em.ivar(Emitter::imod(fixed, n.dims[i]));
      fixed = em.ivar(Emitter::idiv(fixed, n.dims[i]));
      b.len[i] = 1;
    }
  } else {
    for (int64_t i = rank - 1; i > sd; --i) {
      b.lo[i] = em.ivar(Emitter::imod(fixed, n.dims[i]));
      fixed = em.ivar(Emitter::idiv(fixed, n.dims[i]));
      b.len[i] = 1;
    }
  }
  return b;
}

KernelSource lower_literal(const Ctx& c) {
  KernelSource ks;
  ks.strategy = "literal";
  ks.entry = "sfx_lit_" + c.name;
  fill_common(c, ks);
  const Graph& g = c.g;
  const Program& p = c.p;
  // materialised members and their statements
  std::map<int, const Stmt*> mat;
  int64_t max_chunk = 1;
  for (const Stmt& s : p.stmts)
    if (s.kind == SFX_STMT_MATERIALIZE) {
      mat[s.instr] = &s;
      max_chunk = std::max(max_chunk, g.nodes[s.instr].numel() / p.blocks);
    }
  int B = static_cast<int>(std::min<int64_t>(256, std::max<int64_t>(32, (max_chunk + 31) / 32 * 32)));
  Emitter em(g, p, 1, c.wide);
  std::string sig = signature(c, em, ks.entry, B);
  Code body;
  em.code = &body;
  const std::string& it = em.idx_t;
  int64_t staging = 0;  // extra smem for two-phase writes into an aliased buffer
  // ready-set simulation (reference exec.cpp:300-392): arena reads only of
  // members materialised earlier in this block and not overwritten since.
  std::set<int> ready;
  std::set<int> read_now;
  std::string blk = "blk";
  std::map<int, Box> boxes;
  em.resolve = [&](int node, const std::vector<Ix>& comps) -> std::string {
    if (!ready.count(node)) return "";
    read_now.insert(node);
    const Node& n = g.nodes[node];
    const Stmt& s = *mat.at(node);
    Box& b = boxes[node];
    std::vector<Ix> local(comps.size());
    std::string L = "0";
    for (size_t d = 0; d < comps.size(); ++d) {
      std::string off = b.lo[d] == "0" ? comps[d].e : "(" + comps[d].e + "-" + b.lo[d] + ")";
      L = Emitter::iadd(Emitter::imul(L, b.len[d]), off);
      if (!Emitter::is_lit(L)) L = em.ivar(L);
    }
    std::string v = em.fresh("s");
    const char* T = ctype(n.dtype);
    em.code->line(std::string("const ") + T + " " + v + " = ((const " + T + "*)(sfx_arena + " + fmt_i(s.offset) +
                  "))[" + L + "];");
    return v;
  };
  body.line("extern __shared__ __align__(16) unsigned char sfx_arena[];");
  body.line("for (" + it + " blk = blockIdx.x; blk < " + fmt_i(p.blocks) + "; blk += gridDim.x) {");
  body.indent++;
  em.push();
  for (const Stmt& s : p.stmts) {
    if (s.kind == SFX_STMT_BARRIER) {
      body.line("__syncthreads();");
      continue;
    }
    if (s.kind != SFX_STMT_MATERIALIZE) continue;
    const Node& n = g.nodes[s.instr];
    Box b = chunk_box(em, n, s, blk);
    const int64_t chunk = n.numel() / p.blocks;
    const char* T = ctype(n.dtype);
    // detect whether this write aliases a ready buffer it reads (two-phase commit)
    bool shared_dest = s.dest == SFX_DEST_SHARED;
    std::string stage;
    Code saved;
    read_now.clear();
    Code tmp;
    tmp.indent = body.indent + 1;
    Code* outer = em.code;
    // emit the element loop body into tmp first to learn which buffers it reads
    em.code = &tmp;
    em.push();
    std::string k = em.fresh("k");
    std::vector<Ix> local = em.from_linear(em.uni(k), b.len);
    std::vector<Ix> comps(n.rank());
    for (int d = 0; d < n.rank(); ++d) comps[d] = em.uni(em.ivar(Emitter::iadd(b.lo[d], local[d].e)));
    std::string v = em.value(s.instr, comps);
    bool hazard = false;
    if (shared_dest)
      for (int r : read_now) {
        const Stmt& rs = *mat.at(r);
        int64_t len = g.nodes[r].numel() / p.blocks * 4;
        if (rs.offset < s.offset + s.bytes && s.offset < rs.offset + len) hazard = true;
      }
    if (shared_dest) {
      if (hazard) {
        staging = std::max<int64_t>(staging, chunk * 4);
        tmp.line(std::string("((") + T + "*)(sfx_arena + " + fmt_i(p.arena_bytes) + "))[" + k + "] = " + v + ";");
      } else {
        tmp.line(std::string("((") + T + "*)(sfx_arena + " + fmt_i(s.offset) + "))[" + k + "] = " + v + ";");
      }
    } else {
      std::string lin = "0";
      for (int d = 0; d < n.rank(); ++d) lin = Emitter::iadd(Emitter::imul(lin, n.dims[d]), comps[d].e);
      tmp.line("out" + std::to_string(s.root_index) + "[" + lin + "] = " + v + ";");
    }
    em.pop();
    em.code = outer;
    body.line("for (" + it + " " + k + " = threadIdx.x; " + k + " < " + fmt_i(chunk) + "; " + k + " += " +
              std::to_string(B) + ") {");
    body.text += tmp.text;
    body.line("}");
    if (shared_dest && hazard) {
      body.line("__syncthreads();");
      body.line("for (" + it + " " + k + " = threadIdx.x; " + k + " < " + fmt_i(chunk) + "; " + k + " += " +
                std::to_string(B) + ")");
      body.line(std::string("  ((") + T + "*)(sfx_arena + " + fmt_i(s.offset) + "))[" + k + "] = ((" + T +
                "*)(sfx_arena + " + fmt_i(p.arena_bytes) + "))[" + k + "];");
    }
    if (shared_dest) {
      for (auto itr = ready.begin(); itr != ready.end();) {
        const Stmt& rs = *mat.at(*itr);
        int64_t len = g.nodes[*itr].numel() / p.blocks * 4;
        bool overlap = rs.offset < s.offset + s.bytes && s.offset < rs.offset + len;
        if (overlap && *itr != s.instr)
          itr = ready.erase(itr);
        else
          ++itr;
      }
      ready.insert(s.instr);
      boxes[s.instr] = b;
    }
  }
  body.line("__syncthreads();");
  em.pop();
  body.indent--;
  body.line("}");
  ks.code = assemble(sig, body);
  ks.block = B;
  ks.grid_x = std::min<int64_t>(p.blocks, static_cast<int64_t>(kNumSMs) * 16);
  ks.smem = static_cast<int>(p.arena_bytes + staging);
  ks.vector_width = 1;
  ks.note = "reference geometry: blocks=" + std::to_string(p.blocks) + " arena=" + std::to_string(p.arena_bytes) + "B";
  return ks;
}

}  // namespace lw
}  // namespace sfx
