/* SPDX-License-Identifier: Apache-2.0
 *
 * xengine_b200 — C ABI of the B200-native XEngine hot path.
 *
 * The reference (arXiv 2212.09290, /root/reference/proj) is a pure C++20
 * library with no FFI layer; its public API lives in proj/include/xengine/ (one .hpp per module).
 * Every entry point below replaces one reference function (or the inner loop
 * of one) and says which, as file:line under proj/.  The C++ mirror of the
 * reference API (include/xengine/b200.hpp) and the Python bindings
 * (paper_2212_09290_b200/_lib.py) are thin layers over these symbols.
 *
 * Conventions
 *   - Every function returns int status: XE_OK (0), or an xengine::Errc value
 *     + 1 (proj/include/xengine/errors.hpp:9-42), or XE_ERR_CUDA / XE_ERR_NCCL /
 *     XE_ERR_ARG.  xe_last_error() returns the thread-local message.
 *   - No exceptions cross this boundary; plain pointers and sizes only.
 *   - A handle's problem/model data never changes after construction, but
 *     the handle also owns evaluation scratch (best-of-batch partials, the
 *     staging buffers of the canonical/host entry points) and one CUDA
 *     stream: use a handle from one host thread at a time (one handle per
 *     thread or per GPU for concurrency).
 *   - Buffers documented "device" must be device pointers (cudaMalloc / torch
 *     CUDA tensors); "host" buffers may be pageable or pinned.
 */
#ifndef XENGINE_B200_H
#define XENGINE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
  XE_OK = 0,
  /* 1 + xengine::Errc (errors.hpp:9-42) */
  XE_ERR_MALFORMED_DOCUMENT = 1,
  XE_ERR_NON_TOPOLOGICAL_EDGE = 2,
  XE_ERR_UNKNOWN_DEVICE = 3,
  XE_ERR_NON_POSITIVE_SIZE = 4,
  XE_ERR_NEGATIVE_COST = 5,
  XE_ERR_EMPTY_NETWORK = 6,
  XE_ERR_PERCENT_OUT_OF_RANGE = 7,
  XE_ERR_MISSING_LINK = 8,
  XE_ERR_DIMENSION_MISMATCH = 9,
  XE_ERR_INCOMPLETE_ENERGY_TABLE = 10,
  XE_ERR_UNKNOWN_VARIABLE = 11,
  XE_ERR_NON_INTEGRAL_BINARY = 12,
  XE_ERR_EMPTY_SOLUTION = 13,
  XE_ERR_INFEASIBLE_MARKER = 14,
  XE_ERR_INFEASIBLE_PROBLEM = 15,
  XE_ERR_TOO_LARGE = 16,
  XE_ERR_EXTERNAL_SOLVER_UNAVAILABLE = 17,
  XE_ERR_SOLVER_FAILED = 18,
  XE_ERR_UNPARSABLE_SOLUTION = 19,
  XE_ERR_OBJECTIVE_MISMATCH = 20,
  XE_ERR_ILLEGAL_ASSIGNMENT = 21,
  XE_ERR_ILLEGAL_SCHEDULE = 22,
  XE_ERR_EMPTY_SERIES = 23,
  XE_ERR_NON_POSITIVE_TIME = 24,
  XE_ERR_IO = 25,
  /* boundary-only */
  XE_ERR_CUDA = 100,
  XE_ERR_NCCL = 101,
  XE_ERR_ARG = 102,
  XE_ERR_NO_DEVICE = 103
};

/* ---- K2 validity bits --------------------------------------------------
 * One bit per constraint family of check_assignment (model.cpp:430-469) on
 * the completion of (R,S) (model.cpp:471-549); bits 0..14 non-zero <=>
 * check_assignment(build_model(p,opts), complete_assignment(p,opts,R,S))
 * returns a non-empty list.  On a completion only FIXED_ZERO, EQ8, EQ9,
 * EQ11, EQ12, EQ16_HI, ENERGY_* and U_BOUND can fire; the others hold by
 * construction and are listed for completeness. */
enum {
  XE_F_FIXED_ZERO = 1u << 0,   /* R(d,t,i>t) or S(d,t,i>=t) set (model.cpp:126-132) */
  XE_F_EQ8 = 1u << 1,          /* diagonal not on exactly one device */
  XE_F_EQ9 = 1u << 2,          /* total diagonal count != T */
  XE_F_EQ11 = 1u << 3,         /* S(d,t+1,i) > S(d,t,i)+R(d,t,i) */
  XE_F_EQ12 = 1u << 4,         /* computed op with a parent resident nowhere */
  XE_F_EQ13 = 1u << 5,
  XE_F_EQ14 = 1u << 6,
  XE_F_EQ16_LO = 1u << 7,
  XE_F_EQ16_HI = 1u << 8,      /* hazard row (only together with EQ11) */
  XE_F_Z_LINK = 1u << 9,
  XE_F_P_LINK = 1u << 10,
  XE_F_ENERGY_DEV = 1u << 11,
  XE_F_ENERGY_TOTAL = 1u << 12,
  XE_F_U_BOUND = 1u << 13,     /* U > b(1+tol)+tol, tol = 1e-6 (model.cpp:441-445) */
  XE_F_OTHER = 1u << 14,       /* binary / P range / space (never on a completion) */
  XE_F_BUDGET = 1u << 15,      /* integer peak_d > b_d (solver.cpp:237,249; schedule.cpp:181) */
  XE_F_DECODE = 1u << 16,      /* decode() raises IllegalAssignment (schedule.cpp:63-71) */
  XE_F_DECODE_FREED = 1u << 17 /* some copy source was freed earlier in its timestep */
};
#define XE_F_CHECK_MASK 0x7fffu

/* ---- problem ----------------------------------------------------------- */
/* Structure-of-arrays image of xengine::Problem (problem.hpp:18-60) after
 * copy_cost (problem.cpp:358-380) has been applied to every (edge, ds, dc). */
typedef struct xe_problem_desc {
  int32_t D, T, E;
  const int64_t* output_bytes; /* [T] */
  const double* cost_ms;       /* [D][T]  (device-major) */
  const int32_t* edge_src;     /* [E] edge declaration order */
  const int32_t* edge_dst;     /* [E] */
  const double* copy_ms;       /* [E][D][D]; diagonal ignored; NaN = no link covers the copy (MissingLink
                                  when build_model / an evaluator / a charged objective_value copy needs it) */
  const int64_t* budget_bytes; /* [D] */
  /* optional energy model (model.hpp:50-56); has_energy = 0 -> none */
  int32_t has_energy;
  double alpha;
  const double* q_joules;        /* [D][T] */
  const uint8_t* has_dev_limit;  /* [D] */
  const double* dev_limit;       /* [D] */
  int32_t has_total_limit;
  double total_limit;
  double board_joules;
} xe_problem_desc;

typedef struct xe_problem xe_problem; /* opaque; owns device copies */

typedef struct xe_model_opts {
  int32_t strict_free;         /* ModelOptions::strict_free (model.hpp:58-62) */
  int32_t quadratic_objective; /* ModelOptions::quadratic_objective */
  int32_t use_energy;          /* apply the problem's energy model (add_energy_extension) */
} xe_model_opts;

const char* xe_last_error(void);
const char* xe_version(void);

/* Parses a problem document (load_problem, problem.cpp:228-244, including the
 * layered training-graph form, problem.cpp:190-224/280-338) and the optional
 * energy section (parse_energy, model.cpp:314-367) on the host, then uploads. */
int xe_problem_load_json(const char* json_text, int device, xe_problem** out);
/* Host-only parse (no device touched): a handle on which only
 * xe_problem_describe / xe_problem_destroy are valid.  Lets host tooling and
 * CPU tests check the loader without a GPU. */
int xe_problem_parse_json(const char* json_text, xe_problem** out);
/* Uploads an already-resolved problem (validate_problem, problem.cpp:254-278). */
int xe_problem_create(const xe_problem_desc* desc, int device, xe_problem** out);
int xe_problem_destroy(xe_problem* p);
/* Host view of the resolved arrays (pointers stay valid for the handle's life). */
int xe_problem_describe(const xe_problem* p, xe_problem_desc* out);
/* Names of the loaded document (synthesized "d<k>" / "op<i>" for handles built
 * from arrays); NULL for an out-of-range index. */
const char* xe_problem_device_id(const xe_problem* p, int32_t d);
const char* xe_problem_op_name(const xe_problem* p, int32_t i);
/* with_budgets (problem.cpp:382-393): new handle, same problem, new budgets. */
int xe_problem_with_budgets(const xe_problem* p, const int64_t* budgets, xe_problem** out);

/* ---- K1: MILP assembly (build_model, model.cpp:86-312) ------------------ */
typedef struct xe_csr xe_csr; /* opaque; device-resident model */

typedef struct xe_csr_info {
  int64_t n_cols;   /* 4DT^2 + DT(E+T) + TED(D-1) (model.hpp:14-31 order) */
  int64_t n_rows;   /* constraints in emission order */
  int64_t nnz;
  int64_t n_rows_mps; /* rows written to MPS (P_LINK dropped when quadratic) */
  int32_t D, T, E;
  int32_t n_tags;   /* 14 (ConstraintTag, model.hpp:36-39) */
  int64_t tag_rows[16]; /* rows per ConstraintTag */
} xe_csr_info;

/* Device pointers into the model (valid while the handle lives). */
typedef struct xe_csr_view {
  const int64_t* row_ptr; /* [n_rows+1] */
  const int32_t* col;     /* [nnz] column = closed-form VarRef index */
  const double* val;      /* [nnz] */
  const double* rhs;      /* [n_rows] */
  const int8_t* sense;    /* [n_rows] 'L','G','E' */
  const uint8_t* tag;     /* [n_rows] ConstraintTag */
  const int32_t* ordinal; /* [n_rows] per-tag ordinal */
  const double* obj;      /* [n_cols] objective (0 where absent) */
  const uint8_t* obj_present; /* [n_cols] 1 where the reference map holds an entry */
  const double* lb;       /* [n_cols] */
  const double* ub;       /* [n_cols] (FX 0 -> 0, BV -> 1, U -> budget, P -> 1) */
  const uint8_t* kind;    /* [n_cols] 0 fixed-zero, 1 binary, 2 memory(U), 3 product(P) */
} xe_csr_view;

int xe_build_csr(const xe_problem* p, const xe_model_opts* opts, xe_csr** out);
int xe_csr_destroy(xe_csr* m);
int xe_csr_get_info(const xe_csr* m, xe_csr_info* out);
int xe_csr_get_view(const xe_csr* m, xe_csr_view* out);
/* Column-major copy (stable by row) for SpMTV and MPS emission. */
int xe_csr_build_csc(xe_csr* m);
int xe_csr_get_csc(const xe_csr* m, const int64_t** col_ptr, const int32_t** row,
                   const double** val);
/* Bit-exact write_mps (mps_io.cpp:109-199) of the model.  Two-call: pass
 * buf = NULL to get the size in *len, then a buffer of *len bytes. */
int xe_write_mps(xe_csr* m, char* buf, size_t* len);
/* Host copy of the model; any NULL member is skipped.  Sizes from
 * xe_csr_get_info (n_rows + 1 row offsets, nnz entries, n_cols columns). */
typedef struct xe_csr_host {
  int64_t* row_ptr; int32_t* col; double* val; double* rhs; int8_t* sense;
  uint8_t* tag; int32_t* ordinal; double* obj; uint8_t* obj_present;
  double* lb; double* ub; uint8_t* kind;
} xe_csr_host;
int xe_csr_download(const xe_csr* m, const xe_csr_host* out);
/* A model handle from host arrays (a MilpModel the caller built or edited;
 * columns in the closed-form VarRef space of p).  Every xe_csr_host member
 * must be non-NULL; lb/ub/kind/obj/obj_present have n_cols entries. */
int xe_csr_upload(const xe_problem* p, const xe_model_opts* opts, int64_t n_rows, int64_t n_cols,
                  const xe_csr_host* in, xe_csr** out);
/* Row part of check_assignment (model.cpp:449-467) for a dense column vector
 * x (host [n_cols], VarRef order): per row the sequential lhs in term order,
 * scale = max(1, |rhs|, max |term|), violated when the relation's excess
 * exceeds tol*scale.  viol (host [n_rows] or NULL) receives the excess of
 * violated rows and 0 elsewhere; *n_violated the count. */
int xe_check_rows(xe_csr* m, const double* x, double tol, double* viol, int64_t* n_violated);
/* Time of the last K1 assembly (device, CUDA events), milliseconds. */
int xe_csr_last_build_ms(const xe_csr* m, float* ms);

/* ---- K2: batched schedule evaluation ----------------------------------- */
/* Dense cube batch layout ("xe_cube"): candidate-major, per candidate the R
 * cube then the S cube, each [D][T][W] uint32 words with W = ceil(T/32);
 * bit i of row (d,t) is word i>>5, bit i&31.  Replaces BitCube
 * (model.hpp:127-139).  Bytes per candidate: 8*D*T*W. */
size_t xe_cube_bytes(int32_t D, int32_t T);

/* Objective order.  objective_value (model.cpp:369-428) sums its terms
 * sequentially in (d,t,i) then (t,e,dc,ds) order.  The streaming evaluator
 * sums them per timestep: xe_eval_out.obj is that reassociation, within
 * (#terms * 2^-53) relative of the reference (north_star tolerance 1e-6),
 * and bit-identical to it when xe_objective_order_exact() reports 1 (every
 * term dyadic: every partial sum exact in any order).  xe_best.obj/index
 * are always exact: the near-best candidates are re-scored in the
 * reference's order and the first minimum of those bits wins. */
int xe_objective_order_exact(const struct xe_problem* p, int32_t* exact);
/* Per handle: exact != 0 makes every batched evaluation sum each candidate's
 * objective in the reference's order (the reference-order kernels; slower),
 * 0 (default) allows the streaming evaluator's reassociation. */
int xe_problem_set_exact_objective(struct xe_problem* p, int32_t exact);

typedef struct xe_eval_out {
  double* obj;      /* [n] objective_value of the completion (model.cpp:369-428), see above */
  int64_t* peak;    /* [n][D] max_t,v U(d,t,v) = replay peaks (schedule.cpp:326-367) */
  uint32_t* flags;  /* [n] XE_F_* bits */
} xe_eval_out;

typedef struct xe_best {
  double obj;       /* best objective among candidates with (flags & mask) == 0 */
  int64_t index;    /* lowest index attaining it (solver.cpp:57-61 tie rule); -1 none */
  int64_t n_valid;
} xe_best;

/* Evaluates n candidates.  cubes, out arrays: device pointers.  out may have
 * NULL members to skip writing them.  best (host, may be NULL) receives the
 * argmin over candidates whose flags & valid_mask == 0.  stream: a cudaStream_t;
 * NULL is the legacy default stream (as in every CUDA library). */
/* A problem handle owns the staging and scratch buffers of these calls: use a
 * handle from one host thread and on one stream at a time (calls on different
 * streams must be ordered by the caller); open one handle per stream
 * otherwise. */
int xe_eval_cubes(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cubes,
                  int64_t n, xe_eval_out* out, uint32_t valid_mask, xe_best* best,
                  void* stream);
/* Same, host buffers: copies in/out inside the call (the end-to-end path).
 * Host->device copies are pipelined in chunks over two streams; page-locked
 * buffers (cudaHostAlloc / torch pin_memory) are DMA'd directly. */
int xe_eval_cubes_host(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cubes,
                       int64_t n, xe_eval_out* out, uint32_t valid_mask, xe_best* best);

/* Candidate-interleaved layout ("xe_cube_il", T <= 256, D <= 8): the native
 * layout of the lane-per-candidate evaluators.  With NW = ceil(T/64) u64
 * words per bit row, word j of row (which, d, t) of candidate c (which 0 =
 * R, 1 = S; bit i of word j = operator 64j+i) is at
 *     il[((c / 32) * K + ((which * D + d) * T + t) * NW + j) * 32 + c % 32],
 * K = 2*D*T*NW, so a warp reading one word of 32 candidates touches one
 * 256-byte line.  Buffers hold ceil(n/32)*32 candidates (padding lanes are
 * ignored).  xe_eval_cubes / xe_eval_cubes_host transpose canonical cubes
 * into this layout internally. */
size_t xe_cube_il_bytes(int32_t D, int32_t T, int64_t n);
/* canonical device cubes [n] -> interleaved device buffer (xe_cube_il_bytes) */
int xe_cubes_to_il(const xe_problem* p, const uint32_t* cubes, int64_t n, uint64_t* il, void* stream);
/* Evaluates n interleaved device candidates; same outputs as xe_eval_cubes. */
int xe_eval_cubes_il(const xe_problem* p, const xe_model_opts* opts, const uint64_t* il, int64_t n,
                     xe_eval_out* out, uint32_t valid_mask, xe_best* best, void* stream);

/* Placement candidates: dev[n][T] uint8 device per operator (save_all_assignment,
 * solver.cpp:30-42).  policy 0 = save-all (the reference's family),
 * policy 1 = minimal-save (saved only until the last consumer). */
int xe_eval_placements(const xe_problem* p, const uint8_t* dev, int64_t n, int32_t policy,
                       xe_eval_out* out, uint32_t valid_mask, xe_best* best, void* stream);
/* assignment_oracle (solver.cpp:44-75) as a full GPU sweep over D^T
 * placements in odometer order; writes the winning device vector. */
int xe_assignment_oracle(const xe_problem* p, double* best_obj, int32_t* best_dev,
                         int64_t* n_evaluated);

/* ---- single assignments (the map-based reference API) -------------------
 * Dense column vectors x[n_cols] in VarRef order (model.hpp:18-24):
 * R, S, Z [D][T][T]; F [D][T][E+T]; U [D][T][T]; P [T][E][D][D-1]. */
int64_t xe_model_cols(int32_t D, int32_t T, int32_t E);
/* complete_assignment (model.cpp:471-549) of one canonical host cube. */
int xe_complete_cube(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cube, double* x);
/* objective_value (model.cpp:369-428) of any x, same sequential fp64 order. */
int xe_objective_dense(const xe_problem* p, const xe_model_opts* opts, const double* x, double* obj);

/* ---- K3: PDHG LP relaxation -------------------------------------------- */
typedef struct xe_pdhg_opts {
  int32_t max_iters;
  double tol_rel;           /* relative KKT tolerance (default 1e-6) */
  int32_t check_every;      /* iterations between convergence checks (default 64) */
  int32_t verbose;
  const double* lb_override; /* host [n] or NULL (node bounds for B&B) */
  const double* ub_override; /* host [n] or NULL */
} xe_pdhg_opts;

typedef struct xe_pdhg_result {
  double primal_obj, dual_obj;
  double rel_gap, rel_primal_res, rel_dual_res;
  int32_t iters, restarts, status; /* 0 converged, 1 iteration limit */
  double solve_ms;           /* device time, CUDA events */
  double spmv_ms_per_iter;
  /* presolve: columns with the prohibitive cost (>= 1e9, problem.hpp:16) and
   * lower bound 0 are fixed at 0 during the solve; `certified` = 1 when the
   * final duals price every fixed column non-negatively (reduced cost
   * 1e9 - K'y >= 0), i.e. the fixing provably left the LP optimum unchanged */
  int32_t presolve_fixed, certified;
  /* 1 when the half-steps ran on coded entries (<= 256 distinct matrix
   * values: 4 bytes per entry, scaling applied to the vectors), 0 on
   * scaled fp64 values (12 bytes per entry) */
  int32_t coded_entries;
} xe_pdhg_result;

int xe_pdhg_solve(xe_csr* m, const xe_pdhg_opts* opts, xe_pdhg_result* res,
                  double* x_out /* host [n] or NULL */, double* y_out /* host [m] or NULL */);

/* ---- K4: randomized rounding + repair ---------------------------------- */
/* Samples n candidate cubes from LP marginals x (device [n_cols] or NULL for
 * uniform placements): placement from the R(.,t,t) diagonal, minimal-save S,
 * up to `edits` drop-and-recompute edits, all valid for EQ8/11/12 by
 * construction; a fraction `perturb` gets one random bit flip. */
int xe_round_cubes(const xe_problem* p, const double* x_dev, uint64_t seed, int64_t first,
                   int64_t n, int32_t edits, double perturb, uint32_t* cubes_dev,
                   void* stream);
/* Local-search neighbours of one canonical device cube (the incumbent):
 * each is the base with (probability 1/2) one op moved, with its saves, to
 * another device, then up to `edits` drop-and-recompute edits and an
 * optional random bit flip; candidate k a pure function of (seed, first + k). */
int xe_mutate_cubes(const xe_problem* p, const uint32_t* base_dev, uint64_t seed, int64_t first, int64_t n,
                    int32_t edits, double perturb, uint32_t* cubes_dev, void* stream);
/* Local-search neighbours in R space: 1..max_moves random moves on the base's
 * computations R (recompute a parent where one of its consumers is computed;
 * drop a recomputation; move a computation to another device), then the
 * canonical saves of the result: each tensor kept on the device of its latest
 * computation exactly at the steps where it is needed before it is computed
 * again.  max_moves = 0 returns the base's R with its canonical saves.
 * n_base bases (independent local-search chains, device [n_base][cube
 * words]); n a multiple of n_base, candidate k moves base k / (n / n_base).
 * Candidate k is a pure function of (seed, first + k, its base).  T <= 256. */
int xe_move_cubes(const xe_problem* p, const uint32_t* base_dev, int64_t n_base, uint64_t seed, int64_t first,
                  int64_t n, int32_t max_moves, uint32_t* cubes_dev, void* stream);
/* Placement-space neighbours (device buffers): neighbour k copies base
 * k / (n / n_base) ([n_base][T] u8) and moves 1..max_moves random ops to a
 * random device that can run them; a pure function of (seed, first + k). */
int xe_move_placements(const xe_problem* p, const uint8_t* base_dev, int64_t n_base, uint64_t seed, int64_t first,
                       int64_t n, int32_t max_moves, uint8_t* dev_out, void* stream);
/* n uniform random placements dev[n][T] (device buffer): op i on a device
 * that can run it (cost < 1e9), candidate k a pure function of
 * (seed, first + k) — the input family of config 5's placement sweep. */
int xe_random_placements(const xe_problem* p, uint64_t seed, int64_t first, int64_t n, uint8_t* dev_out,
                         void* stream);
/* One iteration of the placement local search's chain control, on the device
 * (all buffers device): `chains` chains, each with `chain_n` scored
 * neighbours nb[chains*chain_n][T] (obj / flags from xe_eval_placements).
 * Per chain: its best neighbour (score = obj when (flags & valid_mask) == 0,
 * else +inf; first index among equals) replaces bases[c] and cur[c] when it
 * improves, or after `stall` iterations without improvement when valid;
 * stalled[c] counts.  Then the lowest cur (first chain among equals)
 * replaces *best / best_dev[T] when strictly lower, ++*improvements.  No
 * host synchronisation. */
int xe_placement_chains_step(const xe_problem* p, const double* obj, const uint32_t* flags, uint32_t valid_mask,
                             const uint8_t* nb, int32_t chains, int32_t chain_n, int32_t stall, uint8_t* bases,
                             double* cur, int32_t* stalled, double* best, uint8_t* best_dev, int32_t* improvements,
                             void* stream);

/* ---- best-schedule search (K1 -> K3 -> K4 -> K2, one native call) ------
 * The GPU counterpart of solve_exact / solve_external (solver.hpp:49-58):
 * LP relaxation (PDHG), LP-guided rounding with canonical saves, exact K2
 * scoring, then a population of R-space local searches (xe_move_cubes).
 * Valid = (flags & valid_mask) == 0.  The rounding incumbent is the first
 * minimum in global index order (solver.cpp:57-61); the local search
 * replaces it only when strictly better.  Sharding: rounding block r of rank
 * k is at global index first + (r*world + k)*n_per_round; the local-search
 * seed is (seed, rank); exchanging the per-rank results is the caller's. */
typedef struct xe_search_opts {
  int64_t n_per_round;   /* rounded candidates per round (default 1<<18) */
  int32_t rounds;        /* default 4 */
  int32_t edits;         /* drop-and-recompute edits per rounded candidate (3) */
  uint64_t seed;         /* default 1 */
  int32_t use_lp;        /* 1: LP-guided rounding, LP bound reported (default 1) */
  double lp_tol;         /* PDHG relative tolerance (1e-6) */
  uint32_t valid_mask;   /* default XE_F_CHECK_MASK | XE_F_BUDGET | XE_F_DECODE */
  int32_t canonical;     /* 1: canonical saves on rounded candidates (default 1; both this and the
                            local search are skipped when a cube does not fit the move kernel) */
  int32_t chains;        /* local-search population (256; 0 = rounding only) */
  int32_t chain_n;       /* neighbours per chain per iteration (1024) */
  int32_t chain_iters;   /* iterations (200) */
  int32_t max_moves;     /* moves per neighbour, 1..max_moves (4) */
  int32_t stall;         /* iterations without improvement before a kick (15) */
  int64_t first;         /* global index of the first rounded candidate (0) */
  int32_t rank, world;   /* candidate sharding (0, 1) */
  int64_t time_limit_ms; /* wall-clock limit (0 = none): later rounding rounds and
                            local-search iterations are skipped once it is spent
                            (SearchLimits::time_limit_ms, solver.hpp:22-25) */
} xe_search_opts;

typedef struct xe_search_result {
  double objective;           /* best valid objective found (inf: none; may be finite with index -1:
                                 the local search reached feasibility from over-budget candidates) */
  double rounding_objective;  /* best rounding candidate alone */
  int64_t index;              /* its global index (-1: no valid candidate) */
  double lp_bound;            /* valid lower bound from the LP duals (NaN without LP; -inf when the
                                 prohibitive-cost presolve is not certified by the duals) */
  int32_t has_lp, lp_certified;
  int64_t n_evaluated, n_valid; /* candidates scored; valid rounding candidates */
  int32_t improvements;       /* local-search improvements of the incumbent */
  int32_t time_limited;       /* 1: the time limit cut the search short */
  double lp_value;            /* PDHG primal objective (the relaxation's value to the tolerance) */
  int32_t lp_converged;       /* 1: PDHG met its tolerance (0: iteration limit) */
  int32_t pad_;
} xe_search_result;

void xe_search_opts_default(xe_search_opts* o);
/* cube_host: [cube words] canonical (R, S) cube of the best schedule, or
 * NULL; peaks_host: [D] its per-device peaks, or NULL. */
int xe_search(const xe_problem* p, const xe_model_opts* opts, const xe_search_opts* so, xe_search_result* res,
              uint32_t* cube_host, int64_t* peaks_host, void* stream);

/* ---- solve_exact (proj/include/xengine/solver.hpp:42-50) -------------------
 * The reference's exact search (proj/src/solver.cpp:101-489: per timestep the
 * new operator on one device, recomputations feeding this timestep's
 * computations, saves of tensors with a later consumer, memory trajectory
 * within budget; optimum under tail_less = (cost, sum R, sum S, bit string),
 * solver.cpp:87-92) as a level-synchronous GPU dynamic program over the same
 * (timestep, saved-set) states.  Requires D*T <= 64 like the reference
 * (XE_ERR_TOO_LARGE otherwise).  Budgets: the handle's (use
 * xe_problem_with_budgets for solve_exact's budget override). */
typedef struct xe_exact_opts {
  int64_t node_limit;     /* SearchLimits::node_limit (< 0: none); nodes = legal
                             (state, computation set) frames expanded */
  int64_t time_limit_ms;  /* SearchLimits::time_limit_ms (< 0: none), checked between launches */
  double upper_bound;     /* search-space cost of a known schedule (prunes; INFINITY: none) */
  int64_t max_states;     /* per timestep (default 1 << 26); beyond it: LimitReached */
} xe_exact_opts;

typedef struct xe_exact_result {
  int32_t status;         /* 0 Optimal, 1 Infeasible, 2 LimitReached (SolveStatus order) */
  int32_t found;          /* 1: cube_host holds the optimal schedule */
  double objective;       /* the search's tail cost (solver.cpp:284, reported as objective_ms); NaN if none */
  int64_t sum_r, sum_s;   /* tail_less keys of the optimum */
  int64_t nodes, states;  /* frames expanded, distinct states kept */
  double ms;              /* wall clock */
} xe_exact_result;

void xe_exact_opts_default(xe_exact_opts* o);
/* cube_host: [xe_cube_bytes(D, T) / 4] canonical (R, S) cube of the optimum
 * (R(d,t,.) = the computation set of t, S(d,t+1,.) = the exit set of t,
 * solver.cpp:426-437), or NULL. */
int xe_solve_exact(const xe_problem* p, const xe_model_opts* opts, const xe_exact_opts* eo,
                   xe_exact_result* res, uint32_t* cube_host, void* stream);

/* ---- schedules: decode / validate / replay (proj/src/schedule.cpp) -------
 * proj/include/xengine/schedule.hpp:15-126.  The executable reading of a
 * schedule, computed on the GPU for a batch (the top-K of an evaluated set):
 * per timestep copies (source: lowest device holding the tensor), the
 * compute, the fired frees, then end-of-timestep drops. */
typedef struct xe_action {
  int32_t kind;  /* ActionKind: 0 Compute, 1 Copy, 2 Free, 3 Drop */
  int32_t timestep, slot;
  int32_t device, op;   /* Compute / Free / Drop (op: Compute / Drop) */
  int32_t src, dst;     /* Copy / Free: edge endpoints (src == dst: a self edge) */
  int32_t from, to;     /* Copy: devices */
} xe_action;

typedef struct xe_decode_error {
  int32_t code;  /* 0 ok; IllegalAssignment: 1 tensor u resident on no device,
                    2 the copy source of u was freed earlier in timestep t (schedule.cpp:57-71) */
  int32_t t, v, u;
} xe_decode_error;

/* decode(complete_assignment(R, S)) of n canonical cubes (host): actions of
 * candidate k in actions[offsets[k] .. offsets[k+1]) (empty when errors[k].code
 * != 0).  actions == NULL: offsets only (size the buffer, call again). */
int xe_decode_cubes(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cubes, int64_t n,
                    int64_t* offsets /* [n+1] */, xe_action* actions, xe_decode_error* errors /* [n] or NULL */);
/* decode of one dense assignment x[n_cols] (VarRef order): R, Z, S, F bits are
 * the assignment's own values > 0.5, as decode reads the map (schedule.cpp:40-129). */
int xe_decode_dense(const xe_problem* p, const double* x, int64_t* n_actions, xe_action* actions,
                    xe_decode_error* error);

typedef struct xe_violation {
  int32_t kind;   /* ViolationKind: 0 ComputeWithoutInputs, 1 CopyFromNonResident,
                     2 BudgetExceeded, 3 FreeNonResident, 4 UncomputedOperator */
  int32_t device, timestep, slot;
  int64_t bytes;  /* BudgetExceeded: occupied bytes at the check */
  int32_t a, b;   /* detail operands: (operator, missing input) | tensor | operator */
} xe_violation;

/* validate (schedule.cpp:131-240) of n action lists (host arrays as from
 * xe_decode_cubes); budgets [D] or NULL (the problem's).  violations == NULL:
 * v_offsets only. */
int xe_validate_schedules(const xe_problem* p, const xe_action* actions, const int64_t* offsets, int64_t n,
                          const int64_t* budgets, int64_t* v_offsets /* [n+1] */, xe_violation* violations);
/* replay (schedule.cpp:261-369) of n LEGAL action lists (run validate first:
 * the reference raises IllegalSchedule): total action cost (NaN when a copy
 * runs along an undeclared edge: the caller prices it with the link model),
 * the Eq. 1 objective rebuilt from availability, the per-slot memory series
 * memory[n][D][T][T] (or NULL) and the per-device peaks [n][D]. */
int xe_replay_schedules(const xe_problem* p, const xe_model_opts* opts, const xe_action* actions,
                        const int64_t* offsets, int64_t n, double* total_ms, double* eq1, int64_t* memory,
                        int64_t* peaks);
/* Text forms (host): format_schedule (schedule.cpp:440-475) and trace_csv
 * (:523-530) with the problem's device ids and operator names.  buf NULL:
 * *len = bytes needed. */
int xe_format_schedule(const xe_problem* p, const xe_action* actions, int64_t n_actions, char* buf, size_t* len);
int xe_trace_csv(const xe_problem* p, const int64_t* memory /* [D][T][T] */, char* buf, size_t* len);
/* parse_schedule (schedule.cpp:477-521): *n_actions in/out (capacity / count). */
int xe_parse_schedule(const xe_problem* p, const char* text, xe_action* actions, int64_t* n_actions);
/* The same with caller-provided names (device_ids [D], op_names [T], the
 * problem name for parse errors; NULL: the handle's). */
int xe_format_schedule_named(const xe_problem* p, const xe_action* actions, int64_t n_actions,
                             const char* const* device_ids, const char* const* op_names, char* buf, size_t* len);
int xe_trace_csv_named(const xe_problem* p, const int64_t* memory, const char* const* device_ids, char* buf,
                       size_t* len);
int xe_parse_schedule_named(const xe_problem* p, const char* text, const char* const* device_ids,
                            const char* const* op_names, const char* problem_name, xe_action* actions,
                            int64_t* n_actions);

/* ---- multi-GPU from the C / C++ host -------------------------------------
 * One xe_ctx per GPU (device, rank, world, NCCL communicator, stream), used
 * by one host thread at a time.  Rank 0 creates the id (xe_nccl_unique_id)
 * and the caller distributes it (MPI, a file, torch.distributed ...).  The
 * candidate sweeps shard with no data-path collective; the exchanges are the
 * incumbent's (all-reduce MIN of the objective bits, MIN of the global index
 * among ranks holding it, SUM of valid counts: the first-minimum rule of
 * solver.cpp:57-61 across ranks) and the winning schedule's broadcast.
 * NCCL is loaded at xe_ctx_create (libnccl.so.2); errors: XE_ERR_NCCL. */
#define XE_NCCL_ID_BYTES 128
typedef struct xe_ctx xe_ctx;
int xe_nccl_unique_id(uint8_t* id /* [XE_NCCL_ID_BYTES] */);
int xe_ctx_create(int device, int rank, int world, const uint8_t* id, xe_ctx** out);
int xe_ctx_destroy(xe_ctx* c);
int xe_ctx_info(const xe_ctx* c, int32_t* device, int32_t* rank, int32_t* world);
/* best: this rank's best-of-batch (index local to its shard) -> the global
 * one; index_offset = the shard's first global index. */
int xe_ctx_exchange_best(xe_ctx* c, int64_t index_offset, xe_best* best);
/* xe_search sharded over the context's ranks (rank/world of so are set from
 * the context): rounding blocks interleaved by rank, one local-search
 * population per rank, the global rounding incumbent, the best final
 * schedule (the rounding incumbent on ties) broadcast to every rank. */
int xe_search_dist(const xe_problem* p, const xe_model_opts* opts, const xe_search_opts* so, xe_ctx* c,
                   xe_search_result* res, uint32_t* cube_host, int64_t* peaks_host);

#ifdef __cplusplus
}
#endif
#endif /* XENGINE_B200_H */
