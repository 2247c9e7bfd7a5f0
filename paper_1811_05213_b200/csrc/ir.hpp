// Internal, index-based view of the reference graph + KernelProgram handed in
// through the C ABI (include/sfx.h).  Mirrors reference proj/include/stitchfuse/
// ir.hpp:82-125 (Instruction/TensorGraph) and kernelgen.hpp:25-54 (KernelProgram).
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "sfx.h"

namespace sfx {

struct Error : std::runtime_error {
  sfx_status code;
  Error(sfx_status c, const std::string& what) : std::runtime_error(what), code(c) {}
};

struct Node {
  std::string id;
  int op = SFX_OP_PARAMETER;
  int kind = 0;
  int dtype = SFX_F32;
  std::vector<int64_t> dims;
  std::vector<int> operands;
  std::vector<int64_t> perm, dim_map, reduce_dims;
  int reducer = SFX_REDUCE_SUM;
  double scalar = 0.0;
  std::vector<double> literal;

  int64_t numel() const {
    int64_t n = 1;
    for (int64_t d : dims) n *= d;
    return n;
  }
  int rank() const { return static_cast<int>(dims.size()); }
  bool is_splat() const { return op == SFX_OP_CONSTANT && literal.size() == 1; }
};

struct Stmt {
  int kind = SFX_STMT_INLINE;
  int instr = -1;
  int64_t split_dim = 0, sword = 1;
  int sched = SFX_SCHED_ROW;
  int dest = SFX_DEST_OUTPUT;
  int64_t offset = 0, bytes = 0;
  int root_index = 0;
};

struct Program {
  std::vector<int> members;  // ascending id
  std::set<int> member_set;
  std::vector<int> roots;    // comp.roots order (ascending id)
  int fusion_root = -1;
  int64_t blocks = 1;
  int block_threads = 64;
  int64_t arena_bytes = 0;
  std::vector<Stmt> stmts;
  std::vector<int> externals;  // operands outside the group, ascending id (splats included)
  std::vector<int> inputs;     // externals minus splat constants = kernel input slots
  // an unfused matmul barrier run as its own kernel (not a planned group;
  // members = roots = {the matmul}, no statements)
  bool barrier = false;
  // read geometry per materialised member (sfx_member_plan; defaults to the
  // member's statement): arena offset and schedule the executor reads with
  struct ReadPlan {
    int64_t offset = -1, split_dim = 0, sword = 1;
    int sched = SFX_SCHED_ROW;
  };
  std::map<int, ReadPlan> reads;
  bool is_member(int n) const { return member_set.count(n) > 0; }
};

struct Graph {
  std::vector<Node> nodes;
  std::vector<int> outputs;
  std::vector<Program> programs;
  std::vector<std::vector<int>> users;  // distinct users per node
};

// Builds and validates the internal graph (shape rules of reference ir.cpp:215-323,
// program structure of kernelgen.cpp:75-104).  Throws sfx::Error.
Graph graph_from_desc(const sfx_graph_desc* desc);

// The reference executor's geometry self-checks (stale arena read, chunk
// containment, overlapping root write, incomplete coverage; exec.cpp:320-327,
// 399, 410), decided at lowering time.  Throws sfx::Error(SFX_ERR_EXEC).
void check_executor_geometry(const Graph& g, const Program& p);

const char* ew_name(int kind);
int ew_arity(int kind);

}  // namespace sfx
