/*
 * kbe200 — C ABI of the B200 (sm_100a) two-time Kadanoff–Baym propagator.
 *
 * The reference (kbesolve 0.1.0, pure Python/numpy) has no FFI layer; its
 * boundary is the Python API re-exported by pkg/src/kbesolve/__init__.py:3-66.
 * Every entry point below replaces one reference operator on the step path
 * (file:line cited per function).  The Python package
 * paper_2505_19467_b200 binds these with ctypes and keeps
 * the reference's names, argument meaning and exception types.
 *
 * Conventions
 *   - complex128 values are `double[2]` pairs (re, im), passed as void*.
 *   - every pointer argument is DEVICE memory unless the name ends in _host.
 *   - every call is asynchronous on the given CUDA stream (`void* stream`,
 *     a cudaStream_t; NULL = legacy default stream) and returns an int status
 *     (KBE_OK = 0); kbe_last_error() describes the last failure.
 *   - nothing allocates device memory: all buffers are owned by the caller
 *     (the Python driver allocates them once, at construction).
 *
 * Packed, time-sliced history layout (one per function; G and Sigma):
 *   hist[k_local][ slice_offset(s) + (b/32)*256 + c*32 + b%32 ]    complex128
 *   slice s holds, for b = 0..s, eight complex planes c:
 *     c = 0..3  the LOWER-triangle block X(t_s, t_b)   (row-major 2x2)
 *     c = 4..7  the UPPER-triangle block Y(t_b, t_s)
 *   G:     lower = G<  (advanced along rows),    upper = G>  (along columns)
 *   Sigma: lower = S>  (selfenergy.py:318),      upper = S<  (selfenergy.py:317)
 *   Everything else follows from X(t',t) = -X(t,t')^dagger (state.py:95-109).
 *   Points are grouped in blocks of 32: one block of one slice (8 planes x 32
 *   points, 4 KB) is contiguous, so the collision stream moves it with ONE bulk
 *   copy.  plane_len(s) = 32*ceil((s+1)/32) padded points per plane.
 */
#ifndef KBE200_H
#define KBE200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KBE_OK 0
#define KBE_ERR_ARG 1
#define KBE_ERR_CUDA 2
#define KBE_ERR_UNSUPPORTED 3

#define KBE_MAX_ITER 16      /* StepConfig.max_iter ceiling on the device path */
#define KBE_MAX_NK 128       /* largest n_k the Sigma kernel takes (kbe_max_n_k()) */
#define KBE_MAX_RANKS 8      /* k-shard ranks of one NVLink/NVSwitch domain (peer-to-peer exchange) */
#define KBE_TILE_B 32        /* collision warp-task: history points            */
#define KBE_TILE_S 32        /* collision tile: time slices (a warp task takes 8, 16 or 32 of them) */
#define KBE_COL_CHUNK 8      /* column-direction partial slots: one per 8 slices */
#define KBE_REPORT_W 32      /* doubles per StepReport row (8 + KBE_MAX_ITER + 8) */

/* Report row layout (doubles):
 *  0 step, 1 iterations, 2 residual, 3 converged, 4 anticommutation drift
 *  (max over local k), 5 sum over local k of n_v + n_c, 6 non-finite flag,
 *  7 sum over local k of Re Tr[h0(k; t_n) rho(k; t_n)] (one-body energy without the
 *  hf term; rho = -i G<(t_n, t_n), h0 = build_h without hartree_fock, model.py:123-152),
 *  8.. residual history (KBE_MAX_ITER entries), then sums over local k of rho_00,
 *  rho_11, Re rho_01, Im rho_01 (the hf energy term needs the global k-mean of rho),
 *  then 4 reserved. */

/* Everything a step needs.  Scalars mirror StepConfig / ModelConfig
 * (propagator.py:44-52, model.py:27-37); pointers are caller-owned device
 * buffers sized by the kbe_*_bytes / kbe_tri_size helpers. */
typedef struct kbe_problem {
    int32_t n_k;          /* global k-point count (even, kgrid.py:30-39)          */
    int32_t k_lo;         /* local k range [k_lo, k_hi) of this rank               */
    int32_t k_hi;
    int32_t n_steps;      /* capacity N: slices 0..N                               */
    int32_t quad;         /* 0 trapezoid, 1 simpson (collision.py:31-61)           */
    int32_t limit_mode;   /* 0 as-printed, 1 langreth (collision.py:188-191, 211-219) */
    int32_t hf;           /* hf_mode == "on"                                       */
    int32_t max_iter;     /* corrector cap, <= KBE_MAX_ITER                         */
    int32_t interacting;  /* any(U != 0): Sigma is evaluated (propagator.py:265)   */
    int32_t nbb;          /* partial-sum columns per output: ceil((N+1)/TILE_B)    */
    int32_t nsb;          /* partial-sum columns per output: ceil((N+1)/KBE_COL_CHUNK) */
    int32_t pad0;
    double dt, eps, dipole_re, dipole_im;
    int64_t tri;          /* complex elements per k of one packed history          */
    void* g_hist;         /* [k_local][tri]                                        */
    void* s_hist;         /* [k_local][tri]                                        */
    const double* eps_v;  /* [n_k] band tables (model.py:71-85), global k          */
    const double* eps_c;
    const double* u_table;/* [N+1] U on the grid (model.py:46-56)                  */
    const double* u_mid;  /* [N+1] U at the step-n midpoint (model.py:59-68)       */
    const double* amp;    /* [N+1] pulse amplitude at the step-n midpoint (88-103) */
    void* row_part;       /* [k_local][nbb][N+1][4] complex: I< row sums, per point chunk */
    void* col_part;       /* [k_local][nsb][N+1][4]: I< row, column-direction sums       */
    void* gc_part;        /* [k_local][nbb][N+1][4]: I> column sums, per point chunk     */
    void* lr_old;         /* [k_local][N+1][4]: I<(t_{n-1}, t_l) kept for the step */
    void* col_old;        /* [k_local][N+1][4]: I>(t_j, t_{n-1}) kept for the step */
    void* front_send;     /* NULL (1 rank) or one all-gather chunk: [k_local][slice of capacity N] + 16-complex control tail */
    void* front_all;      /* NULL (1 rank) or [ranks][chunk] (gathered)                */
    void* ctl;            /* kbe_ctl_bytes() of device control state               */
    double* reports;      /* [N+1][KBE_REPORT_W]                                   */
    void* phi;            /* [N+1][k_local][4] complex: Cayley propagator per step */
    /* limit_mode = langreth only (NULL otherwise): I> rows and I< columns are
     * accumulated separately; the G pass also scatters along columns. */
    void* row_part_g;     /* [k_local][nbb][N+1][4]: I> row sums                    */
    void* col_part_g;     /* [k_local][nsb][N+1][4]: I> column-direction sums       */
    void* lc_part;        /* [k_local][nbb][N+1][4]: I< column, row-direction sums  */
    void* gc_part_c;      /* [k_local][nsb][N+1][4]: I> column, column-direction    */
    void* lc_part_c;      /* [k_local][nsb][N+1][4]: I< column, column-direction    */
    /* incremental collision evaluations (as-printed; NULL g_sh disables them): a
     * repeated evaluation at the same frontier whose vectors moved by <= 1e-7 since the
     * last full one writes M_fp32 * (v - v_prev) into delta slots instead of
     * re-streaming M in FP64. */
    void* g_sh;           /* [k_local][tri] complex64 shadow of the final G slices   */
    void* s_sh;           /* [k_local][tri] complex64 shadow of the final Sigma slices */
    void* v_prev;         /* [k_local][2][8*plane_len(N)]: G and Sigma frontier of the last full evaluation */
    void* fcol_part;      /* [k_local][N+1][4]: column-direction sums of the frontier slice */
    void* row_delta;      /* incremental evaluations' M_fp32 dv (complex64), shapes of row_part, */
    void* col_delta;      /* col_part and gc_part; K3 adds them to the full evaluation's  */
    void* gc_delta;       /* partials while the last evaluation was incremental          */
    void* i_red;          /* [2][k_local][N+1][4]: I< rows (+ the diagonal) reduced by K3a (split K3); */
    void* g_red;          /* I> columns likewise; [1] = the base sums of the last full evaluation  */
    /* peer-to-peer exchange over NVLink (p2p_world > 1; front_send / front_all are
     * then unused except for the initial slice): every rank owns a kbe_p2p_bytes()
     * buffer, opened by every peer through kbe_p2p_export / kbe_p2p_open. */
    int32_t p2p_world;    /* ranks exchanging through peer memory (0/1: off)       */
    int32_t p2p_rank;
    void* p2p_local;      /* this rank's buffer                                    */
    void* p2p_peers[KBE_MAX_RANKS];  /* every rank's buffer as mapped here (incl. self) */
} kbe_problem;

/* ---- layout helpers (host-callable, no device work) ---------------------- */
int      kbe_abi_version(void);
int64_t  kbe_plane_len(int32_t s);
int64_t  kbe_slice_offset(int32_t s);              /* in complex elements      */
int64_t  kbe_tri_size(int32_t n_steps);            /* complex elements per k    */
int64_t  kbe_ctl_bytes(void);
int64_t  kbe_sizeof_problem(void);
const char* kbe_last_error(void);

/* ---- state (state.py) --------------------------------------------------- */
/* init_state ground state (state.py:56-87): zero both histories, then
 * G<(0,0) = i diag(1,0), G>(0,0) = -i diag(0,1) per local k; resets ctl. */
int kbe_init_history(const kbe_problem* p, void* stream);

/* ---- Sigma (selfenergy.py) ---------------------------------------------- */
/* evaluate_sigma_batched (selfenergy.py:261-325): both components of the
 * second-Born Sigma on the step-n frontier, all n+1 pairs, local k, one
 * launch; writes Sigma slice n.  `it` >= 1 makes the call a no-op once the
 * corrector has converged (device-side convergence, see kbe_update). */
int kbe_sigma_frontier(const kbe_problem* p, int32_t n, int32_t it, void* stream);

/* sigma_slice / polarizability / sigma_first / sigma_second
 * (selfenergy.py:59-236) on batch-last (n_k,2,2,nb) buffers.  Any of
 * pol_out, s1_out, s2_out, sigma_out may be NULL.  If pol_in is non-NULL it
 * replaces the computed polarizability in the first term (sigma_first's pol
 * argument).  u1, u2: [nb] doubles.  Outputs cover k in [k_lo, k_hi)
 * (pol_out always covers all n_k). */
int kbe_sigma_slice(int32_t n_k, int32_t nb, const void* g_primary, const void* g_reversed,
                    const double* u1, const double* u2, int32_t k_lo, int32_t k_hi,
                    const void* pol_in, void* pol_out, void* s1_out, void* s2_out,
                    void* sigma_out, void* stream);

/* ---- collision integrals (collision.py) ---------------------------------- */
/* collision_frontier (collision.py:228-277) at step n into the partial-sum
 * workspace: row sums over the Sigma history triangle (slices 0..n) and the
 * column sums over the G history triangle (slices 0..n-1).  Ordered after all
 * earlier work on the stream (only the step sequencer overlaps it with Sigma). */
int kbe_collision_frontier(const kbe_problem* p, int32_t n, int32_t it, void* stream);

/* collision_row (collision.py:141-162): the kernel-level row-slice contraction on
 * caller buffers (device, complex128, C order): dg_first (n_k,2,2,T1), g_first
 * (n_k,2,2,T2); s_like, s_other (n_k,2,2,T,P); w1 (T1), w2 (T2) with T1, T2 <= T,
 * or, when w2_matrix != 0, w2 (T,P) and T2 = T; out (n_k,2,2,P) = term1 + term2. */
int kbe_collision_row(int32_t n_k, int32_t T, int32_t P, int32_t T1, int32_t T2, int32_t w2_matrix,
                      const void* dg_first, const void* g_first, const void* s_like, const void* s_other,
                      const double* w1, const double* w2, void* out, void* stream);

/* Reduce the partials of the last kbe_collision_frontier(n) into the four
 * CollisionSlice arrays (collision.py:165-176), local k, batch-last:
 * lesser_row/greater_row (k_local,2,2,n+1), lesser_col/greater_col (k_local,2,2,n). */
int kbe_collision_slice(const kbe_problem* p, int32_t n, void* lesser_row, void* greater_row,
                        void* lesser_col, void* greater_col, void* stream);

/* ---- predictor / corrector (propagator.py) -------------------------------- */
/* phase 0: predict_frontier + _write_frontier (propagator.py:138-163, 208-212)
 * phase 1: correct_frontier + _frontier_residual + _write_frontier
 *          (propagator.py:166-220), corrector iteration `it` (0-based).
 * The Cayley propagator (propagator.py:77-94) is built in-kernel from
 * h(k; t_{n-1/2}) (model.py:123-152). */
int kbe_update(const kbe_problem* p, int32_t n, int32_t phase, int32_t it, void* stream);

/* k-mean of rho for hf_mode="on" (model.py:106-120): phase 0 uses
 * rho(t_{n-1}), phase 1 uses (rho(t_{n-1}) + rho(t_n))/2.  Local k sum;
 * the caller all-reduces across ranks before dividing (kbe_hf_finalize). */
int kbe_hf_mean(const kbe_problem* p, int32_t n, int32_t phase, int32_t it, void* stream);

/* Phi(t_{n-1/2}) for local k into p->phi[n] after the host has all-reduced the
 * hf k-sum across ranks (hf_mode="on" with k-shards; one rank does this inside
 * kbe_hf_mean).  The table for hf_mode="off" is built by kbe_init_history. */
int kbe_build_phi(const kbe_problem* p, int32_t n, int32_t it, void* stream);

/* End of step n: observables_at / anticommutation_drift (state.py:125-137),
 * _frontier_finite (propagator.py:223-226), StepReport row into reports[n].
 * A non-finite frontier poisons the device state: later calls are no-ops. */
int kbe_finish_step(const kbe_problem* p, int32_t n, void* stream);

/* One whole PropagationDriver.step() (propagator.py:316-382) on one rank:
 * Sigma(n-1), I(n-1), predictor, max_iter x (Sigma(n), I(n), corrector), finish
 * (kbe_sigma_frontier, kbe_collision_frontier, kbe_update, kbe_finish_step). */
int kbe_step(const kbe_problem* p, int32_t n, void* stream);

/* Steps n_first..n_last (inclusive) back to back (PropagationDriver.run,
 * propagator.py:384-392).  use_graph = 0: kbe_step per step (converged corrector
 * iterations launch as no-ops).  use_graph != 0 (one rank only): one CUDA graph per
 * problem, replayed per step with its kernel nodes' arguments rewritten; corrector
 * iterations 1..max_iter-1 sit behind IF conditional nodes that the previous
 * iteration's update kernel enables only while the residual is > eps, so nothing
 * is launched after convergence.  Results are bitwise identical either way. */
int kbe_run(const kbe_problem* p, int32_t n_first, int32_t n_last, int32_t use_graph, void* stream);

/* Speculative iteration counts (PropagationDriver.run, one rank): steps n_first..n_last
 * launching only m <= max_iter corrector iterations each.  A step still unconverged
 * after m sets the control block's needs_more word (offset kbe_ctl_needs_more_offset())
 * to its index and every later launch becomes a no-op; kbe_resume_step(n, m) clears
 * the word and runs iterations m..max_iter-1 and the finish of step n, after which the
 * host continues from n+1.  Results equal kbe_run's bitwise. */
int kbe_run_iters(const kbe_problem* p, int32_t n_first, int32_t n_last, int32_t m, void* stream);
int kbe_resume_step(const kbe_problem* p, int32_t n, int32_t m_done, void* stream);
int64_t kbe_ctl_needs_more_offset(void);
/* Byte offset of the hf_mode="on" k-sum of rho (4 complex) in the control block: the
 * k-sharded host all-reduces exactly these bytes between kbe_hf_mean and kbe_build_phi. */
int64_t kbe_ctl_hf_sum_offset(void);
/* Kernels one evaluation launches on the stream path (Sigma, collision, [hf], [K3a],
 * update): the launch count the bench reports.  -1 on an invalid problem. */
int kbe_launches_per_eval(const kbe_problem* p);
/* Sigma kernel variant for every later K1 launch of this process (env KBE_SIGMA, read
 * by the driver): 0 auto (FFT for power-of-two n_k > 2, the correlations at n_k = 2, DMMA DFT
 * GEMMs otherwise), 1 FFT,
 * 2 DMMA DFT GEMMs, 3 the O(n_k^2) correlation kernel.  Returns the previous setting,
 * -1 for an unknown kind.  Replaces nothing in the reference: its sigma_second
 * (selfenergy.py:139-203) has one algorithm; this selects how K1 computes the same Sigma. */
int kbe_set_sigma_variant(int32_t kind);
/* KBE_MAX_NK: the driver validates n_k against it before allocating anything. */
int32_t kbe_max_n_k(void);

/* Drop the step graph cached for this problem's control block (driver teardown). */
int kbe_release(const kbe_problem* p);

/* ---- peer-to-peer frontier exchange (k-sharded ranks) ---------------
 * Replaces the per-iteration NCCL all-gather (propagator.py's _gather_frontier) by
 * stores from the update kernel into every peer's buffer over NVLink plus epoch
 * flags.  Buffer = [2 parities][world][chunk complex] + world flags + epoch + watchdog, where
 * chunk = k_local * 8 * plane_len(N) + 16 (slice + control tail). */
int64_t kbe_p2p_bytes(const kbe_problem* p, int32_t world);
/* cudaMalloc + zero a buffer and export its IPC handle (64 bytes) for the peers. */
int kbe_p2p_alloc(int64_t bytes, void** ptr_out, void* ipc_handle_out);
/* Map a peer's buffer from its IPC handle (cudaIpcOpenMemHandle); close with kbe_p2p_close. */
int kbe_p2p_open(const void* ipc_handle, void** ptr_out);
int kbe_p2p_close(void* ptr);
int kbe_p2p_free(void* ptr);
/* Synchronous 8-byte device read (the exchange buffer's watchdog word: nonzero = a
 * peer wait timed out, value - 1 = the rank waited for). */
int kbe_p2p_read_u64(const void* dev_ptr, void* host_out);
/* Publish this rank's send chunk (front_send: the initial slice) to every peer at the
 * next epoch; used after kbe_init_history instead of the NCCL all-gather. */
int kbe_p2p_publish(const kbe_problem* p, void* stream);

/* ---- layout conversion (TwoTimeGF / SigmaHistory accessors) -------------- */
/* Rebuild the reference layout (k_local,2,2,N+1,N+1) of one function from the
 * packed history: which = 0 -> lower-stored (G<, S>), 1 -> upper-stored (G>, S<).
 * Entries beyond slice `frontier` are zero. */
int kbe_unpack(const void* hist, int64_t tri, int32_t k_local, int32_t n_steps, int32_t frontier,
               int32_t which, void* out, void* stream);
/* Retarded function of the packed G history in the reference layout:
 * G^R(t,t') = theta(t-t') [G>(t,t') - G<(t,t')], theta(0) = theta0 on the diagonal
 * (theta0 = 1: the t -> t'+ limit, G^R(t,t) = -i up to the anticommutation drift).
 * A derived accessor (SURVEY finding 2: the reference has no G^R); its parity follows
 * from G< / G> parity.  Entries with t < t' or beyond slice `frontier` are zero. */
int kbe_unpack_retarded(const void* hist, int64_t tri, int32_t k_local, int32_t n_steps, int32_t frontier,
                        double theta0, void* out, void* stream);
/* Inverse: pack slices 0..frontier of a reference-layout pair (lower-stored,
 * upper-stored) into a packed history (zeroing nothing else). */
int kbe_pack(const void* lower_full, const void* upper_full, int32_t k_local, int32_t n_steps,
             int32_t frontier, int64_t tri, void* hist, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KBE200_H */
