// Expression emitter: turns "value of member X at multi-index I" into SSA CUDA
// source, with memoisation (CSE across lanes/phases), index algebra for
// broadcast / transpose / reshape / bitcast, and 128-bit load coalescing.
//
// This is the device-code twin of the reference's recursive inliner
// eval_element + compute_element (reference proj/src/exec.cpp:141-213,
// 312-343): thread composition becomes straight-line register code, external
// reads become (vectorised) global loads, and strategies override how
// materialised members are obtained (registers, shared memory, combined
// reductions) through `resolve`.
#pragma once

#include <functional>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "ir.hpp"

namespace sfx {

// One component of a multi-index, for the lane currently being emitted.
//   UNI : same value for every lane of the vector
//   PLUS: lane-0 value `base` (a multiple of the vector width) + lane
//   CPLX: lane-dependent, not affine in the lane
enum IxKind { IX_UNI = 0, IX_PLUS = 1, IX_CPLX = 2 };
struct Ix {
  std::string e;
  std::string base;
  int kind = IX_UNI;
};

struct Code {
  std::string text;
  int indent = 1;
  void line(const std::string& s) {
    text.append(static_cast<size_t>(indent) * 2, ' ');
    text += s;
    text += '\n';
  }
};

std::string fmt_f32(double v);   // exact hex-float literal of (float)v
std::string fmt_f64(double v);   // exact hex-float literal of v
std::string fmt_i(int64_t v);
const char* ctype(int dtype);

class Emitter {
 public:
  Emitter(const Graph& g, const Program& p, int vec, bool wide_index);

  const Graph& g;
  const Program& p;
  int V;          // lanes per vector (1 or 4)
  int lane = 0;   // lane being emitted
  std::string idx_t;
  Code* code = nullptr;
  std::map<int, std::string> input_ptr;  // external node -> kernel parameter
  std::set<int> streaming;               // externals read once (no-L1-allocate loads)
  // externals staged in shared memory for the current row: node ->
  // (const float* smem pointer variable, linear index of the row's first element)
  std::map<int, std::pair<std::string, std::string>> staged;
  // externals staged as a transposed shared-memory tile: element at input comps
  // c lives at arr[B - b0][A - a0], B = c[jb] (or c[jb] % mb when that dim
  // merges several root axes), A = c[ja] (or c[ja] / sa % ma)
  // swz: the vectorised tile instead — a flat [64 a][64 b] array, rows along
  // the root's innermost axis a, 16-byte chunks of b XOR-swizzled by (a/4)&7:
  // element (a, b) at arr[a*64 + (((b>>2) ^ ((a>>2)&7))<<2) + (b&3)], written
  // with 128-bit stores and read conflict-free by 8 a-rows x 4 b per warp
  struct Tile {
    std::string arr, b0, a0;
    int jb = 0, ja = 0;
    int64_t mb = 0, sa = 1, ma = 0;
    bool swz = false;
  };
  std::map<int, Tile> tiled;
  // Strategy hook for member nodes: return a variable name to use instead of
  // evaluating the member's op, or "" to evaluate it inline.
  std::function<std::string(int node, const std::vector<Ix>& comps)> resolve;
  // Divisions by a reduction-dependent value (softmax's e / sum) through the
  // divisor's IEEE reciprocal (<= 1 ulp from the quotient; such outputs carry
  // the reduction-order tolerance anyway).  Off in the literal tier, which
  // keeps the reference's arithmetic.
  bool rcp_reduced_divisors = false;

  std::string value(int node, const std::vector<Ix>& comps);

  // index algebra
  Ix lane_plus(const std::string& base);  // PLUS component for the current lane
  Ix uni(const std::string& e) { return Ix{e, e, IX_UNI}; }
  std::vector<Ix> from_linear(const Ix& lin, const std::vector<int64_t>& dims);
  Ix linearize(const std::vector<Ix>& comps, const std::vector<int64_t>& dims);
  std::string ivar(const std::string& expr);

  // integer expression helpers with constant folding
  static bool is_lit(const std::string& s, int64_t* v = nullptr);
  static std::string imul(const std::string& a, int64_t k);
  static std::string iadd(const std::string& a, const std::string& b);
  static std::string idiv(const std::string& a, int64_t k);
  static std::string imod(const std::string& a, int64_t k);

  std::string fresh(const char* prefix);
  void push();
  void pop();
  std::string find(const std::string& key) const;
  void bind(const std::string& key, const std::string& var);

  // Reduce-fold expression used by the sequential (reference-order) fold.
  std::string seq_fold(int reducer, int dtype, const std::string& acc, const std::string& v);
  // Elementwise expression for node n with operand values.
  std::string ew_expr(const Node& n, const std::vector<std::string>& a);

  // statistics
  int loads_vec = 0, loads_scalar = 0;

 private:
  std::string load(int node, const std::vector<Ix>& comps);
  std::string staged_load(int node, const std::vector<Ix>& comps);
  std::string reduce_loop(int node, const std::vector<Ix>& comps);
  std::string dot_loop(int node, const std::vector<Ix>& comps);
  bool reduce_dependent(int node);
  std::map<int, bool> reduce_dep_;
  std::vector<std::map<std::string, std::string>> scopes_;
  int next_ = 0;
};

}  // namespace sfx
