/*
 * planeq_witness.h -- C-ABI of the sm_100a stage-discharge engine.
 *
 * This boundary replaces the reference's per-stage discharge:
 *   pkg/src/planeq/stages.py:267  run_stage(plan, stage, solver_argv, timeout_s)
 * and the pieces it drives:
 *   pkg/src/planeq/ops.py:923     sym_execute      (symbolic execution of both sub-DFGs)
 *   pkg/src/planeq/smt.py:318     SolverSession.check  (SMT decision of residual pairs)
 *   pkg/src/planeq/stages.py:221  _confirm          (replay of a candidate countermodel)
 *
 * Instead of symbolic expressions plus an SMT query, every stage is compiled
 * (on the host, in C++) from a flat tensor-op program into straight-line
 * scalar bytecode over the prime field F_p, p = 2^31 - 1, and evaluated on the
 * GPU for a batch of random witness assignments; uninterpreted functions
 * (EXP, RSQRT, SIGMOID) are keyed hash functions F_p -> F_p. A stage is
 * refuted iff some valid witness makes an obligation's two sides differ; the
 * failing witness is an exact integer counterexample.
 *
 * All entry points return 0 on success and a negative PQW_E* code on failure;
 * pqw_last_error() describes the last failure on the calling thread. An engine
 * is not thread-safe: call it from one thread at a time (it parallelises its
 * own compilation internally). Engines on different devices are independent.
 * The library's parallel loops share one pool of host threads (PQW_THREADS
 * caps them) that stay parked between calls; a loop started while another
 * holds the pool, or in a forked child, runs on threads of its own.
 * No torch types cross this boundary: plain pointers and sizes only.
 */
#ifndef PLANEQ_WITNESS_H
#define PLANEQ_WITNESS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQW_ABI_VERSION 5
#define PQW_PRIME 2147483647u /* 2^31 - 1 */

/* error codes */
#define PQW_OK 0
#define PQW_EINVAL (-1)   /* malformed program / argument */
#define PQW_ENODEV (-2)   /* no CUDA device or driver */
#define PQW_ECUDA (-3)    /* CUDA runtime failure */
#define PQW_ESTATE (-4)   /* call out of order (e.g. run before compile) */
#define PQW_EPLAN (-5)    /* plan not well formed: the host's own checks raise the
                             reference's exception for it (pqw_plan_* only) */

/* per-stage compile status (pqw_stage_add out_status[0]) */
#define PQW_STAGE_OK 0            /* residual obligations go to the GPU            */
#define PQW_STAGE_PROVEN 1        /* every obligation closed by value numbering   */
#define PQW_STAGE_REFUTED_CONST 2 /* constant/int obligation differs; info = obl   */
#define PQW_STAGE_PAR_DIV0 3      /* parallel side divides by a constant zero      */
#define PQW_STAGE_LOG_DIV0 4      /* logical side divides by a constant zero       */
#define PQW_STAGE_BAD_INDEX 5     /* embedding id outside its table                 */
#define PQW_STAGE_PENDING 6       /* pqw_stage_add: not compiled yet (pqw_stage_status) */
#define PQW_STAGE_LOSSY 7         /* an exact constant is a nonzero multiple of p: the
                                     field image loses it, the stage stays undecided */

/* tensor-op program opcodes (pqw_stage_add ir stream) */
enum pqw_top {
  PQW_T_VARS = 1,      /* out <- fresh variables; attr: var-table offset           */
  PQW_T_INTS = 2,      /* out <- integer constants; attr: const-table offset        */
  PQW_T_SLICE = 3,     /* out <- in[lo.. lo+out.shape]; attrs: lo per axis          */
  PQW_T_RESID = 4,     /* out <- in0 - sum(in1..)  (last partial member)            */
  PQW_T_CHECK = 5,     /* obligations in0[i] == in1[i]; attr: first obligation id   */
  PQW_T_CHECKSUM = 6,  /* obligations in0[i] == sum_k ink[i]; attr: first obl id   */
  PQW_T_SIDE = 7,      /* attr: 0 = logical ops follow, 1 = parallel ops follow     */
  PQW_T_ADD = 16, PQW_T_SUB, PQW_T_MUL, PQW_T_DIV, PQW_T_DROPOUT, PQW_T_SILU_GRAD,
  PQW_T_IDENTITY, PQW_T_SCALE, PQW_T_SHIFT, PQW_T_POW, PQW_T_RSQRT, PQW_T_SILU,
  PQW_T_MOVE, PQW_T_SOFTMAX, PQW_T_CREATE_MASK, PQW_T_APPLY_MASK, PQW_T_VIEW,
  PQW_T_TRANSPOSE, PQW_T_EXPAND, PQW_T_SUM, PQW_T_MEAN, PQW_T_MATMUL, PQW_T_EINSUM,
  PQW_T_FULL, PQW_T_CHUNK, PQW_T_EMBEDDING, PQW_T_EMBEDDING_GRAD, PQW_T_GNORM_SQ,
  PQW_T_ALL_REDUCE, PQW_T_ALL_GATHER, PQW_T_REDUCE_SCATTER, PQW_T_ALL_TO_ALL
};

/*
 * Stage-program opcodes (what the GPU interprets; see pqw_stage_bytecode and
 * paper_2506_15961_b200/csrc/isa.hpp). A program is a table of per-warp stream
 * offsets followed by one instruction stream per warp; an instruction is a
 * header record {op | fn << 8 | k << 16, n, aux, 0} and payload records that
 * list, 8 ops at a time, the u32 fields of n independent ops of one kind.
 */
enum pqw_bop {
  PQW_B_END = 0,
  PQW_B_DOT,    /* d = sum_j a_j * b_j over k pairs (k = 1: multiply)        */
  PQW_B_SUM,    /* d = sum_j a_j over k terms (k = 2: add)                    */
  PQW_B_SUB, PQW_B_NEG,
  PQW_B_HASH,   /* d = f_fn(a): keyed hash standing in for EXP/RSQRT/SIGMOID */
  PQW_B_INV,    /* d_i = a_i^-1, batched (one inversion per instruction)      */
  PQW_B_VAR,    /* d = witness value of a stage variable                      */
  PQW_B_CONST,
  PQW_B_CHK,    /* obligation: lhs == rhs                                     */
  PQW_B_DEN,    /* definedness: a != 0                                        */
  PQW_B_FILL, PQW_B_SPILL, /* global spill slot <-> shared value file         */
  PQW_B_WAIT,   /* wait for other warps' progress                             */
  PQW_B_SIGNAL, /* publish this warp's progress                               */
  PQW_B_NUM_OPS
};

/* One 16-byte record of a stage program (header or payload). */
typedef struct pqw_ins {
  uint32_t op;  /* header: op | fn << 8 | k << 16; payload: field word 0 */
  uint32_t dst; /* header: n (ops in the bundle);   payload: field word 1 */
  uint32_t a;   /* header: aux (SIGNAL value);      payload: field word 2 */
  uint32_t b;   /* header: 0;                       payload: field word 3 */
} pqw_ins;

/* entries of pqw_image_stats */
#define PQW_IMAGE_STATS_LEN (16 + PQW_B_NUM_OPS)

typedef struct pqw_engine pqw_engine;

/* ABI version (PQW_ABI_VERSION) -- lets the host refuse a stale library. */
int pqw_abi_version(void);

/* Human-readable description of the last error on this thread. */
const char* pqw_last_error(void);

/* Number of visible CUDA devices (0 when no driver/device), never fails. */
int pqw_device_count(void);

/*
 * Create an engine bound to `device`. `seed` keys the witness stream;
 * `fn_keys[3]` key the uninterpreted functions EXP, RSQRT, SIGMOID
 * (host-derived from seed, see paper_2506_15961_b200/field.py).
 * Compilation works without a device; run/probe need one.
 */
int pqw_engine_create(int device, uint64_t seed, const uint64_t fn_keys[3],
                      pqw_engine** out);
void pqw_engine_destroy(pqw_engine* e);

/*
 * Add one stage's tensor-op program (stream layout documented in
 * paper_2506_15961_b200/stages.py). consts: n_consts triples
 * (residue, exact_num, exact_den) -- exact_den == 0 marks an inexact constant.
 * var_keys: per-variable 64-bit keys. Identical programs are recognised here
 * (they compile once); the compilation itself is deferred and runs, spread over
 * host threads, at the first pqw_stage_status / pqw_upload / inspection call.
 * out_status[0] = PQW_STAGE_PENDING, out_status[13] = variables.
 * Returns the stage index (>= 0) or a negative error (malformed header).
 */
int pqw_stage_add(pqw_engine* e, const int32_t* ir, size_t ir_len,
                  const int64_t* consts, size_t n_consts,
                  const uint64_t* var_keys, size_t n_vars, int64_t out_status[16]);

/*
 * Compile status of a stage (compiles every pending stage first):
 * out_status[0] = PQW_STAGE_*, out_status[1] = info (obligation id for
 * REFUTED_CONST / BAD_INDEX), out_status[2] = obligation count, out_status[3] =
 * obligations closed by value numbering, out_status[4] = residual obligations,
 * out_status[7] = max numerator degree of a residual obligation (saturating),
 * out_status[8..9] = lhs/rhs residues of the REFUTED_CONST obligation,
 * out_status[10..11] = their exact integer values (INT64_MIN when not an exact
 * integer), out_status[13] = variables; once the GPU program exists (after
 * pqw_upload): out_status[5] = program records, out_status[6] = shared-memory
 * slots, out_status[12] = field ops per witness, out_status[14] = global spill
 * slots, out_status[15] = instruction bundles.
 */
int pqw_stage_status(pqw_engine* e, int stage, int64_t out_status[16]);

/* Restrict scheduling and upload to the stages flagged in `active` (one flag
 * per queued stage; default: all). Front ends still run for every stage, so a
 * multi-GPU host can cost every stage once and schedule only its share. */
int pqw_stage_select(pqw_engine* e, const uint8_t* active, size_t n);

/* Device cost of a stage after the compiler front end (compiles every pending
 * front end first): scheduling units of its residual cones, 0 for a stage
 * decided at compile time. Negative on error. */
int64_t pqw_stage_cost(pqw_engine* e, int stage);

/* Drop every compiled stage (device image included). */
int pqw_reset(pqw_engine* e);

/* Copy out the compiled bytecode of a stage (for inspection / CPU tests).
 * Returns the instruction count; copies min(count, cap) instructions. */
long pqw_stage_bytecode(pqw_engine* e, int stage, pqw_ins* out, size_t cap,
                        uint32_t* n_slots);

/* Variables in the cone of obligation `obl` of `stage` (sorted var ids);
 * returns the count, copies at most cap. */
long pqw_obligation_support(pqw_engine* e, int stage, uint32_t obl,
                            uint32_t* out, size_t cap);

/* Upload all compiled stages as one device image (plus result buffers). */
int pqw_upload(pqw_engine* e);

/*
 * Evaluate every uploaded GPU stage on witnesses [0, n_witness) on `stream`
 * (a cudaStream_t, NULL = legacy default). Asynchronous; results are read
 * with pqw_results after a stream sync (pqw_results syncs).
 */
int pqw_launch(pqw_engine* e, uint32_t n_witness, void* stream);

/*
 * Per-stage results of the last launch (arrays of length n_stages).
 * first_bad = (witness << 32) | obligation of the smallest failing witness
 * (UINT64_MAX when none); n_valid = witnesses with every denominator nonzero;
 * n_bad = valid witnesses with at least one failing obligation.
 */
int pqw_results(pqw_engine* e, uint64_t* first_bad, uint32_t* n_valid,
                uint32_t* n_bad, size_t n_stages);

/*
 * Re-evaluate one stage at one witness and report both sides of obligation
 * `obl` plus the values of the stage's variables (var_vals, length n_vars of
 * that stage, may be NULL).
 */
int pqw_probe(pqw_engine* e, int stage, uint32_t witness, uint32_t obl,
              uint32_t* lhs, uint32_t* rhs, uint32_t* var_vals, size_t n_vars);

/*
 * Confirm a refutation on the host the way the reference does before it
 * reports one (pkg/src/planeq/stages.py:221-264 _confirm). Re-runs the
 * stage's front end, then:
 *  1. out[0] = the first residual obligation whose cone holds no uninterpreted
 *     function (EXP/RSQRT/SIGMOID or a constant folded from one) and whose
 *     sides differ in F_p at `witness` (all definedness conditions holding
 *     there): an exact rational counterexample, no replay needed; -1: none.
 *  2. Otherwise the real-valued replay: for each of the n_env variable
 *     assignments (env_vals: n_env rows of the stage's variables, in order),
 *     every definedness condition must hold (|v| > 1e-12, v > 1e-12 where the
 *     reference requires positivity), then each residual obligation with an
 *     uninterpreted function in its cone is evaluated in double precision
 *     with the genuine exp, 1/sqrt and logistic functions (a failed
 *     evaluation skips the obligation, as a raised exception does there);
 *     out[1] = the first environment in which some obligation's sides differ
 *     by more than tol, out[2] = that obligation, sides[0..1] = its sides
 *     (out[1] = out[2] = -1: not confirmed).
 * out[3] = residual obligations with an uninterpreted function in their cone.
 */
int pqw_confirm(pqw_engine* e, int stage, uint32_t witness, const double* env_vals,
                size_t n_env, double tol, int64_t out[4], double sides[2]);

/* Device time of the last launch in milliseconds (CUDA events on the launch stream). */
int pqw_last_launch_ms(pqw_engine* e, float* ms);

/* Totals over the compiled GPU stages (PQW_IMAGE_STATS_LEN entries):
 * out[0] = stages on the GPU, out[1] = program records, out[2] = max shared
 * slots of a stage, out[3] = shared slots of the uploaded value file,
 * out[4 + op] = ops of each pqw_bop, out[4 + N] = records of the uploaded
 * image after sharing identical programs, out[5 + N] = compile-cache hits,
 * out[6 + N .. 10 + N] = field ops per witness by class (multiplies, adds,
 * keyed hashes, inversions, compares), out[11 + N] = max global spill slots
 * of a stage, out[12 + N] = bundles, out[13 + N] = cross-warp waits,
 * out[14 + N] = bytes the last pqw_upload copied to the device, out[15 + N] =
 * bytes pqw_results reads back (N = PQW_B_NUM_OPS). Only stages selected by
 * pqw_stage_select count. */
int pqw_image_stats(pqw_engine* e, uint64_t* out, size_t cap);

/* Measured integer-pipe ceiling of this device: field ops per second of
 * register-resident, decode-free kernels: out[0] = F_p multiplies, out[1] =
 * F_p adds, out[2] = keyed-hash evaluations, out[3] = inversions. The
 * roofline denominator of the interpreter (bench.py). */
int pqw_peak_fieldops(int device, double out[4]);


/* ---------------------------------------------------------------------------
 * Native plan core: stage construction and lowering behind the C-ABI.
 *
 * Replaces, for the verify pipeline, the host-side work the reference does
 * per plan and per stage before any decision is taken:
 *   pkg/src/planeq/shapes.py:35-45   validate_concrete (shape rule per node)
 *   pkg/src/planeq/stages.py:79-88   entry_order
 *   pkg/src/planeq/stages.py:91-138  build_stages (lineage-cut backward slices)
 *   pkg/src/planeq/graph.py:96-150   topo_sort (tie-break: device, seq, id)
 *   pkg/src/planeq/stages.py:144-176 + :267-340  interface construction and
 *                                    obligations of run_stage
 * A plan is handed over once as flat arrays (names as NUL-terminated UTF-8
 * strings, resolved here); stages are lowered into the same tensor-op
 * programs pqw_stage_add takes (paper_2506_15961_b200/stages.py lower_stage
 * emits the identical stream) on host threads and queued into an engine.
 * Anything not well formed returns PQW_EPLAN: the caller's own host checks
 * then raise the reference's exception with the reference's message.
 * ------------------------------------------------------------------------- */

/* One dataflow graph. Strings are concatenations of NUL-terminated names. */
typedef struct pqw_graph_desc {
  int64_t n_tensors;
  const char* tensor_names;    /* n_tensors names (graph.tensors order)            */
  const int32_t* tensor_ndim;  /* rank per tensor                                  */
  const int64_t* tensor_dims;  /* concatenated shapes                              */
  const uint8_t* tensor_flags; /* bit 0: dtype "int"; bit 1: meta.enum == "position" */
  int64_t n_nodes;
  const char* node_ids;        /* n_nodes ids (graph.nodes order)                  */
  const int32_t* node_kind;    /* pqw_top opcode of the kind, -1 = unknown kind    */
  const int32_t* node_nin;     /* inputs per node                                  */
  const int32_t* node_nout;    /* outputs per node                                 */
  const char* node_inputs;     /* all input names, node-major                      */
  const char* node_outputs;    /* all output names, node-major                     */
  const int32_t* node_nattr;   /* encoded attribute words per node (see stages.py) */
  const int64_t* node_attrs;   /* concatenated                                     */
  const int32_t* node_device;  /* -1 = None                                        */
  const int64_t* node_seq;
  int64_t n_inputs;
  const char* input_names;     /* graph.inputs                                     */
  /* byte length of each names buffer above (through its last NUL), or 0 when
   * the caller does not know it (the library then scans for the n-th NUL) */
  int64_t tensor_names_len, node_ids_len, node_inputs_len, node_outputs_len, input_names_len;
} pqw_graph_desc;

/* Lineage: checkpoint entries (dict order) and their shards. */
typedef struct pqw_lineage_desc {
  int64_t n_entries;
  const char* logical_names;   /* logical tensor id per entry                      */
  const uint8_t* mode;         /* 0 = full, 1 = partial, 2 = anything else         */
  const int32_t* n_shards;     /* shards per entry                                 */
  const char* shard_names;     /* parallel tensor per shard, entry-major           */
  const int32_t* shard_ndim;   /* ranges per shard                                 */
  const int64_t* ranges;       /* (lo, hi) pairs, concatenated                     */
} pqw_lineage_desc;

typedef struct pqw_plan pqw_plan;

/* Copy a plan in. consts: n_consts triples (residue, exact_num, exact_den) --
 * the plan's distinct rational attributes (scale factor, shift addend, full
 * value), referenced from node_attrs by index. */
int pqw_plan_create(const pqw_graph_desc* logical, const pqw_graph_desc* parallel,
                    const pqw_lineage_desc* lineage, const int64_t* consts, size_t n_consts,
                    pqw_plan** out);
void pqw_plan_destroy(pqw_plan* p);

/* Structural checks and the concrete shape rule of every node of both graphs
 * (validate_concrete). PQW_EPLAN when anything is off. */
int pqw_plan_validate(pqw_plan* p);

/* validate_lineage (graph.py:227-252) as counts: out[0] = hard problems
 * (unknown tensors, bad mode, shard shape != range extents), out[1] = entries
 * whose shard ranges do not tile the logical shape. Any nonzero: the host's
 * validate_lineage produces the reference's messages. */
int pqw_plan_check_lineage(pqw_plan* p, int64_t out[2]);

/* build_stages: out[0] = stages, out[1] = uncovered logical nodes, out[2] =
 * uncovered parallel nodes. PQW_EPLAN when stage construction would raise
 * (it does not require pqw_plan_validate: the reference builds the stages of
 * a reduced plan without re-validating it). */
int pqw_plan_build_stages(pqw_plan* p, int64_t out[3]);

/* Stage `stage`: target (logical tensor index, graph.tensors order). */
int pqw_plan_stage_target(pqw_plan* p, int stage);

/* Node indices of a stage's logical (side 0) or parallel (side 1) slice in
 * the stage's topological order; side 2 / 3: its logical / parallel boundary
 * tensors (Stage.l_inputs / p_inputs, sorted by name). Returns the count,
 * copies at most cap. */
long pqw_plan_stage_nodes(pqw_plan* p, int stage, int side, int32_t* out, size_t cap);

/* Nodes owned by no stage (side 0 logical, 1 parallel), sorted by id. */
long pqw_plan_uncovered(pqw_plan* p, int side, int32_t* out, size_t cap);

/* Lower the stages listed in `stages` (n of them; NULL = all, in order) with
 * variables keyed by `seed` and queue them into `e` (pqw_stage_add). out_index
 * (length n) receives each stage's engine index, or PQW_EPLAN for a stage whose
 * lowering raises in the reference (the host re-lowers it to raise). Lowering
 * runs on host threads (PQW_THREADS caps them). */
int pqw_plan_add_stages(pqw_plan* p, pqw_engine* e, uint64_t seed, const int32_t* stages,
                        size_t n, int32_t* out_index);

/* The tensor-op program of one stage (what pqw_plan_add_stages queues): lens[0]
 * = ir words, lens[1] = const triples, lens[2] = variables; copies what fits. */
int pqw_plan_stage_program(pqw_plan* p, int stage, uint64_t seed, int32_t* ir, size_t ir_cap,
                           int64_t* consts, size_t consts_cap, uint64_t* var_keys,
                           size_t vk_cap, int64_t lens[3]);

#ifdef __cplusplus
}
#endif
#endif /* PLANEQ_WITNESS_H */
