/* CPU numeric oracle for the redsynth-b200 executor.
 *
 * TEST INFRASTRUCTURE ONLY — "the checker". Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it. The product
 * path (paper_2110_10548_b200) never links or calls this code.
 *
 * What it restates: the data-level meaning of the reference's collective
 * rules (/root/reference/proj/src/semantics.cc:203-310) folded over a
 * LoweredProgram exactly as RunLowered folds them
 * (/root/reference/proj/src/dsl.cc:142-164), with
 *   row r of an N-element device buffer = elements [floor(rN/K), floor((r+1)N/K))
 * (the reference's own byte model, simulator.cc:179-181).
 *
 * Numeric contract (fixed so the GPU path can be bit-exact):
 *   - sums run over the group's members in the order the step lists them
 *     (ascending physical id for every synthesized program);
 *   - f32: IEEE single adds left to right, acc = x0 + x1 + ... + x_{n-1};
 *   - bf16: every term widened to f32, summed as above, rounded to bf16
 *     (round-to-nearest-even) once, at the store;
 *   - i32: two's-complement wrapping adds;
 *   - copies (AllGather, Broadcast) move raw bits; Broadcast overwrites every
 *     row the root holds on every member.
 *
 * Parity pinning: the boolean layer (held rows, violations, failing step) is
 * computed by the same premises as the reference and is checked against the
 * reference's own RunLowered (oracle/_ref) by tests/test_oracle.py on every
 * synthesized program of configs 1-3; the arithmetic is pinned by the
 * order-independent int32 identity (final device i = sum over its reduction
 * group) and committed golden vectors (tests/golden/).
 */
#ifndef REDSYNTH_ORACLE_NUMERIC_H_
#define REDSYNTH_ORACLE_NUMERIC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_F32 = 0, ORACLE_BF16 = 1, ORACLE_I32 = 2 };

/* Executes a lowered program in place over K host buffers of `elems`
 * elements each. Program encoding (CSR, same as redsynth_exec.h):
 *   step_op[s]               Collective enum value (semantics.h order)
 *   step_group_ptr[s..s+1]   range of groups of step s
 *   group_member_ptr[g..g+1] range of members of group g in `members`
 * Returns 0 on success; 3 (INVALID_ARGUMENT) for malformed input or an empty
 * step; 9 (FAILED_PRECONDITION) on a rule violation, with *fail_step and
 * *fail_violation (RuleViolation enum value) set. `held_out`, when non-null,
 * receives the final held-row masks: held_out[d*K + r] = column bitmask.
 * K must be <= 64. nthreads <= 0 means "all hardware threads". */
int oracle_execute(int K, int num_steps, const int32_t* step_op, const int32_t* step_group_ptr,
                   const int32_t* group_member_ptr, const int32_t* members, size_t elems,
                   int dtype, void* const* bufs, int nthreads, int* fail_step,
                   int* fail_violation, uint64_t* held_out);

/* Boolean layer only (no buffers): same return codes as oracle_execute. */
int oracle_check(int K, int num_steps, const int32_t* step_op, const int32_t* step_group_ptr,
                 const int32_t* group_member_ptr, const int32_t* members, int* fail_step,
                 int* fail_violation, uint64_t* held_out);

int oracle_hardware_threads(void);

#ifdef __cplusplus
}
#endif

#endif /* REDSYNTH_ORACLE_NUMERIC_H_ */
