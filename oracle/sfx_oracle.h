/* TEST INFRASTRUCTURE — CPU parity oracle.  Not part of the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * A plain-C restatement of the reference's dense op-by-op interpreter
 * `interpret` (reference proj/src/exec.cpp:249-268) and its scalar semantics
 * `compute_element` / `apply_unary` / `apply_binary` / `reduce_fold`
 * (exec.cpp:14-100, 141-229), over the same flat graph descriptor the device
 * library takes (include/sfx.h).  Parity pinned: tests/test_oracle.py checks
 * it bit-for-bit against the reference library itself (oracle/_ref/ref_tool,
 * built from /root/reference) on the committed random-graph and config
 * fixtures (FNV-1a hashes of the reference's outputs in tests/golden/) and on
 * the reference's own known-answer tests (test_exec.cpp:26-106).
 *
 * mode 0: reference semantics (fp32 ops, glibc libm, sequential row-major
 *         folds initialised by the first element) — bit-exact to `interpret`.
 * mode 1: fp64 restatement (every f32 op evaluated in double, reductions
 *         accumulated in double, rounded to f32 at the end) — the yardstick for
 *         the "reduction-order differences allowed" tolerance.
 */
#ifndef SFX_ORACLE_H
#define SFX_ORACLE_H

#include "../include/sfx.h"

#ifdef __cplusplus
extern "C" {
#endif

/* values[i] points to a caller-owned buffer of numel(instr i) 4-byte elements.
 * Parameter buffers are inputs; every other buffer is written.  Returns 0 on
 * success, nonzero (with a message in sfx_oracle_error()) otherwise. */
int sfx_oracle_interpret(const sfx_graph_desc* g, void* const* values, int mode);
const char* sfx_oracle_error(void);
uint64_t sfx_oracle_fnv1a(const void* data, uint64_t n, uint64_t h);
void sfx_oracle_gen(uint64_t seed, uint64_t tensor_index, int is_i32, float lo, float hi, void* out, int64_t n,
                    int64_t offset);

#ifdef __cplusplus
}
#endif
#endif
