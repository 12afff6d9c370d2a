/*
 * tcqr.h -- C ABI of libtcqr.so: TensorCore mixed-precision recursive Gram-Schmidt QR and
 * R-preconditioned CGLS least squares on NVIDIA B200 (sm_100a).  arXiv 1912.05508.
 *
 * Method:
 *   - Alg. 2 "Recursive Modified Gram-Schmidt QR" (Eq. (5) :313-318): split the
 *     columns, recurse left, R12 = Q1'*A2 (line 8), recurse on A2 - Q1*R12 (line 9). Both products
 *     run as FP16-input / FP32-accumulate tcgen05 tensor-core GEMMs ("We use TensorCore to
 *     accelerate these matrix-matrix multiplications") at split nodes wider than
 *     the cutoff (128, Alg. 2 line 3); below it in FP32.
 *   - panelQR: the communication-avoiding MGS panel of Eq. (6) built from
 *     Alg. 4 "256x32 Modified Gram-Schmidt QR" blocks.
 *   - Alg. 5 "CGLS with RMGSQR as Preconditioner", corrected as in
 *     DESIGN.md reading R-A10, with the stop/restart rule R-A11/R-A12.
 *
 * Conventions (all entry points):
 *   - Matrices are COLUMN-MAJOR: element (i, j) of an m x n matrix X with leading dimension ldx
 *     lives at X[i + j*ldx].  A is FP32 problem data (reading R-A14); b and x are FP64.
 *   - Every pointer argument is a DEVICE pointer on the context device, owned by the caller; the
 *     library never frees or retains it after the call returns.  Exception: tcqr_lls_solve_host /
 *     tcqr_factor_host take HOST pointers (end-to-end entry points that include the copies).
 *   - Base pointers must be 16-byte aligned (the FP16 shadows the TMA reads are library-owned,
 *     so any lda >= m is accepted; the component GEMM entry points need FP16 lds % 8 == 0).
 *   - All calls enqueue on the context stream (tcqr_init) and synchronize on it once at the end
 *     to read the device status, so outputs are ready when the call returns.
 *   - Multi-GPU (row partition, one process per GPU): every rank calls with ITS OWN row block
 *     (m = local rows, contiguous in rank order, each >= 32) and identical n, config, tol, maxit.
 *     R and x are replicated bitwise on all ranks.
 *
 * Return codes (LAPACK style; identical on all ranks):
 *     0      success (a CGLS solve that stops at maxit also returns 0 with info->converged = 0,
 *            SPEC.md:324-325 "converged=false (not an error)")
 *    -i      argument i is invalid (1-based position in the C signature)
 *    +k      numerical breakdown at global column k (1-based): zero or non-finite column norm
 *            after orthogonalization, or a non-finite entry in input column k
 *    TCQR_ERR_CUDA / _NCCL / _OOM / _NOT_INIT  (below)
 */
#ifndef TCQR_H_
#define TCQR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCQR_ERR_CUDA (-1001)
#define TCQR_ERR_NCCL (-1002)
#define TCQR_ERR_OOM (-1003)
#define TCQR_ERR_NOT_INIT (-1004)
#define TCQR_ERR_UNSUPPORTED (-1005)

/* Library configuration.  All ranks must pass identical values. */
typedef struct tcqr_config {
  int cutoff;        /* recursion cutoff c: split nodes wider than c use FP16 tensor cores
                        (Alg. 2 line 3; default 128; multiple of 32, >= 32)     */
  int panel_rows;    /* CAQR block rows br (PAPER.md:441-442 uses 256 on V100; default 1024 on
                        B200, reading R-A6; 64..1024, multiple of 32)                        */
  int col_scaling;   /* 1: per-column power-of-two FP16 range guard (reading R-A4; default 1) */
  int restart;       /* 1: FP64 target, one CGLS restart from the true residual (R-A12)        */
  double tol2;       /* restart-pass tolerance (default 1e-8, R-A12 as calibrated on this path)*/
  int stag_window;   /* stagnation window W (default 10, R-A11)                                */
  double stag_floor; /* stagnation floor relative to pass 1's ||s0|| (default 1e-11, R-A11)    */
  int use_graphs;    /* 1: capture the factorization into a CUDA graph and replay (default 1)  */
  int reorth;        /* 1: re-orthogonalize (NEXT-1): factor Q1 again,
                        Q <- Q2, R <- R2 * R1; used by tcqr_factor and tcqr_lls_solve (default 0,
                        i.e. Alg. 5 with the single RMGSQR R)                                  */
  int warm_start;    /* 1: tcqr_lls_solve starts CGLS from the direct QR solution
                        x0 = R^-1 Q' b (Alg. 1; NEXT-2) instead of x0 = 0
                        (Alg. 5 line 4); pass 1 then iterates on r0 = b - A x0 (default 0)      */
  int leaf_kernel;   /* 1: every leaf (w <= min(cutoff, 128), one GPU, m <= 148 * 256) runs as ONE
                        cooperative launch with 256-row blocks resident in shared memory and the
                        Eq. (6) stack factored through its FP64 Gram matrix (reading R-B1);
                        0: one pipelined MGS-root panel launch per 32 columns plus FP32
                        projection launches (default 1).  Across ranks (P > 1): 1 = replicated
                        leaves when P * (rows per rank, padded) fit one such grid (the leaf's rows
                        allgathered, every rank factors the whole leaf, keeps its rows of Q),
                        else the per-leaf TSQR (local leaf, allgather of the P local R's, the
                        stack's leaf, Q_r <- Q_r S_r); 2 = always the per-leaf TSQR             */
  int fp16_split;    /* 1: error-compensated FP16 split for the tensor-core split nodes (NEXT-4,
                        SURVEY.md 8(f); beyond the paper, whose related work on tensor-core
                        precision is PAPER.md:758): X diag(s) = Xh + Xl with Xh = fl16(X diag(s)),
                        Xl = fl16(X diag(s) - Xh); R12 = Q1h'A2h + Q1h'A2l + Q1l'A2h and
                        A2 -= Q1h R12h + Q1h R12l + Q1l R12h (three MMAs each, lo*lo dropped).
                        3x the tensor-core work; opt-in (default 0)                              */
} tcqr_config_t;

/* Per-solve report (SPEC.md:296-299 CglsReport). */
typedef struct tcqr_lls_info {
  int iterations;        /* total CGLS iterations over all passes                      */
  int iterations_pass1;  /* iterations of pass 1                                       */
  int outer_passes;      /* 1 or 2                                                     */
  int converged;         /* 1 if the last pass stopped by tolerance or stagnation      */
  int stop_reason;       /* 0 tol, 1 stagnation, 2 maxit, 3 zero right-hand side       */
  double s0;             /* ||s_0|| of pass 1                                          */
  double final_rel;      /* last pass: best ||s_k|| / ||s_0||                          */
  double qr_ms;          /* device time of the factorization (CUDA events)             */
  double cgls_ms;        /* device time of the CGLS passes                             */
} tcqr_lls_info_t;

/* Create the per-process context on `device`, enqueueing on `cuda_stream` (a cudaStream_t;
 * NULL = legacy default stream).  nccl_unique_id: NULL for one GPU, else a pointer to the
 * 128-byte ncclUniqueId that rank 0 created with tcqr_nccl_unique_id() and broadcast; rank /
 * nranks as in ncclCommInitRank.  Re-initialization finalizes the previous context first. */
int tcqr_init(int device, void* cuda_stream, const void* nccl_unique_id, int rank, int nranks);

/* Write a fresh ncclUniqueId (128 bytes) into `out`.  Returns 0 or TCQR_ERR_NCCL. */
int tcqr_nccl_unique_id(void* out);

/* Destroy the context: frees library-owned workspace, destroys the NCCL communicator. */
int tcqr_finalize(void);

/* Default configuration. */
void tcqr_default_config(tcqr_config_t* cfg);
/* Set the configuration (validated; returns -1 on an invalid field). */
int tcqr_set_config(const tcqr_config_t* cfg);

/* Workspace: op = 0 factor, 1 lls_solve.  bytes receives the device workspace the call needs
 * for an m x n problem (m = local rows).  tcqr_set_workspace hands the library caller-owned
 * device memory (e.g. a torch tensor); when none is set (or it is too small) the library
 * allocates its own with cudaMalloc and keeps it until tcqr_finalize. */
int tcqr_workspace_size(int64_t m, int64_t n, int op, size_t* bytes);
int tcqr_set_workspace(void* dptr, size_t bytes);

/*
 * tcqr_factor -- A = Q R by Alg. 2 / Eq. (6) / Alg. 4 with FP16 tensor-core trailing updates.
 *   m, n  : rows (this rank's rows at P > 1) and columns; need sum_r m_r >= n >= 1, m >= 1.
 *   A     : FP32 m x n column-major, leading dimension lda >= m; read only.
 *   Q     : FP32 m x n output, leading dimension m (row-partitioned like A).  Q == A is allowed
 *           when lda == m (the factorization then runs in place).
 *   R     : FP32 n x n output, leading dimension n: upper triangular, diag(R) > 0, strictly lower
 *           triangle zeroed, replicated on all ranks.
 * Errors: -1 m, -2 n, -3 A, -4 lda, -5 Q, -6 R; +k breakdown at column k.
 */
int tcqr_factor(int64_t m, int64_t n, const float* A, int64_t lda, float* Q, float* R);

/*
 * tcqr_lls_solve -- min_x ||A x - b||_2 (Eq. (1)) by tcqr_factor's R and the
 * corrected Alg. 5.  A is not modified (the factorization runs on a workspace copy; Q is not
 * produced, reading R-A25).
 *   b     : FP64, m entries (this rank's rows);  x : FP64, n entries (replicated output).
 *   tol   : pass-1 threshold on ||s_k|| / ||s_0|| (> 0);  maxit : iteration cap per pass (>= 1).
 *   info  : optional report (may be NULL).
 * Errors: -1 m, -2 n, -3 A, -4 lda, -5 b, -6 x, -7 tol, -8 maxit; +k breakdown in the QR.
 */
int tcqr_lls_solve(int64_t m, int64_t n, const float* A, int64_t lda, const double* b, double* x,
                   double tol, int maxit, tcqr_lls_info_t* info);

/*
 * tcqr_qr_solve -- the direct QR solve x = R^-1 (Q' b) of Alg. 1 lines 3-4 (PAPER.md:187-198,
 * Eq. (4); NEXT-2), with Q and R from tcqr_factor (or any thin QR).
 *   Q : FP32 m x n (ldq >= m; this rank's rows);  R : FP32 n x n upper triangular (ldr >= n);
 *   b : FP64 m (this rank's rows);  x : FP64 n output (replicated).  Device pointers.
 * Q' b is an FP64-accumulated GEMV (allreduced over ranks); R^-1 is applied as the FP64
 * explicit inverse of tcqr_trinv (reading R-A13).  Errors: -1 m, -2 n, -3 Q, -4 ldq, -5 R,
 * -6 ldr, -7 b, -8 x; +k if R(k,k) is zero or not finite.
 */
int tcqr_qr_solve(int64_t m, int64_t n, const float* Q, int64_t ldq, const float* R, int64_t ldr,
                  const double* b, double* x);

/* Host-pointer variants (end-to-end: the H2D copy of A, b and the D2H copy of the result happen
 * inside the call; A, b, Q, R, x are HOST pointers; pinned memory is used if the caller's is). */
int tcqr_factor_host(int64_t m, int64_t n, const float* A, int64_t lda, float* Q, float* R);
int tcqr_lls_solve_host(int64_t m, int64_t n, const float* A, int64_t lda, const double* b,
                        double* x, double tol, int maxit, tcqr_lls_info_t* info);

/* ---------------------------------------------------------------------------------------------
 * Component entry points (the individual hot-path kernels, for parity tests of each §8(a) step).
 * All pointers are device pointers; all enqueue on the context stream and synchronize.
 * ------------------------------------------------------------------------------------------- */

/* K1 (§8a a1, reading R-A4): Xh = fl16(X diag(s)), s_j = 2^-floor(log2 max_i |X_ij|) (s_j = 1 if
 * scaling is 0 or the column is zero); inv_s[j] = 1/s_j.  X FP32 m x w (ldx), Xh FP16 bits
 * (uint16) m x w (ldh).  Returns +j (1-based) for the first column holding a non-finite entry. */
int tcqr_cast_scale(int64_t m, int64_t w, const float* X, int64_t ldx, uint16_t* Xh, int64_t ldh,
                    float* inv_s, int scaling);

/* K3 (§8a a4, Alg. 2 line 8): C (h x w2, ldc, FP32) = A1h' * A2h * diag(col_mult), tcgen05
 * kind::f16 with FP32 accumulation in TMEM, deterministic split-K over the m rows.
 * A1h: FP16 m x h (lda1), A2h: FP16 m x w2 (lda2); col_mult may be NULL (= 1). */
int tcqr_gemm_tn(int64_t m, int64_t h, int64_t w2, const uint16_t* A1h, int64_t lda1,
                 const uint16_t* A2h, int64_t lda2, float* C, int64_t ldc, const float* col_mult);

/* K4 (§8a a5, Alg. 2 line 9 argument): C (m x w2, ldc, FP32) -= (Qh * Bh) * diag(col_mult),
 * Qh FP16 m x h (ldq, MN-major operand), Bh FP16 h x w2 (ldb, K-major operand). */
int tcqr_gemm_nn_update(int64_t m, int64_t h, int64_t w2, const uint16_t* Qh, int64_t ldq,
                        const uint16_t* Bh, int64_t ldb, float* C, int64_t ldc,
                        const float* col_mult);

/* K2 (§8a a3): CAQR-MGS panel (Eq. (6) with Alg. 4 blocks of br rows), w <= 32 columns, in
 * place on X (m x w, ldx); R (w x w, ldr) upper triangular output; br in [64, 1024]. */
int tcqr_panel_qr(int64_t m, int64_t w, float* X, int64_t ldx, float* R, int64_t ldr, int br);

/* K6 helper (Alg. 5 lines 12/18): Minv (n x n FP64, ldm) = R^-1 for upper-triangular FP32 R. */
int tcqr_trinv(int64_t n, const float* R, int64_t ldr, double* Minv, int64_t ldm);

/* K5 (Alg. 5 lines 12/18): y = A v (trans = 0, A m x n) or y = A' v (trans = 1); A FP32, v/y FP64. */
int tcqr_gemv(int trans, int64_t m, int64_t n, const float* A, int64_t lda, const double* v,
              double* y);

/* ---------------------------------------------------------------------------------------------
 * Profiling: per-kernel-class device time (CUDA events recorded on the launching stream around
 * every launch group) with the ALGORITHMIC flops and bytes of each launch.
 * While enabled, CUDA-graph replay is bypassed.  tcqr_profile_enable clears the accumulators;
 * tcqr_profile_read synchronizes and returns the totals for one class.
 * ------------------------------------------------------------------------------------------- */
enum {
  TCQR_COPY = 0,        /* input validation + copy A -> working Q                 */
  TCQR_K1_CAST = 1,     /* K1 FP16 range guard + cast (A2 and final Q columns)    */
  TCQR_K3_TN = 2,       /* K3 tcgen05 R12 = Q1' A2 (split-K + reduction)          */
  TCQR_K3_FINALIZE = 3, /* R12 -> R, scaled FP16 copy of R12                       */
  TCQR_K4_NN = 4,       /* K4 tcgen05 A2 -= Q1 R12                                 */
  TCQR_K2_MGS = 5,      /* K2 CAQR level: Alg. 4 MGS on every row block            */
  TCQR_K2_APPLY = 6,    /* K2 Eq. (6) step 4: Q_b <- Q_b Q_red[b]                  */
  TCQR_K2B_TN = 7,      /* FP32 R12 below the cutoff                               */
  TCQR_K2B_NN = 8,      /* FP32 update below the cutoff                            */
  TCQR_K5_GEMV = 9,     /* CGLS A t and A' r                                       */
  TCQR_K6_TRI = 10,     /* CGLS inv(R) p and inv(R') v                             */
  TCQR_K7_SCALAR = 11,  /* CGLS scalar / vector recurrences                        */
  TCQR_TRINV = 12,      /* one-time explicit inverse of R                          */
  TCQR_K2_LEAF = 13,    /* K2L whole-leaf kernel: panels + FP32 projections (k_leaf.cu) */
  TCQR_NUM_CLASSES = 14
};
int tcqr_profile_enable(int on);
int tcqr_profile_read(int cls, double* ms, double* flops, double* bytes, int* launches);
/* Kernels launched by the most recent graph-replayed tcqr_factor (kernel nodes of its graph). */
int tcqr_last_launch_count(void);

/* Collectives (allreduce / allgather) enqueued by the calling context's most recent
 * tcqr_factor or tcqr_lls_solve (0 at one rank). */
int tcqr_last_collective_count(void);

/* ---------------------------------------------------------------------------------------------
 * Virtual ranks (test seam): the row-partitioned multi-GPU path of tcqr_factor /
 * tcqr_lls_solve / tcqr_qr_solve run by P ranks inside ONE process on ONE device.  Each rank is a
 * host thread with its own context (tcqr_init_virtual binds it to the calling thread; every
 * tcqr_* call from that thread uses it; tcqr_finalize destroys it).  The collectives are the same
 * calls in the same order as with NCCL (Eq. (6) with the ranks as the top tree level,
 * PAPER.md:414-440, reading R-A26; R12 / A'r / ||q||^2 allreduces), carried out through the group's
 * device staging slots: every rank combines the P contributions in rank order, so results are
 * bitwise identical across ranks.  Each virtual rank's grids use 1/P of the SMs.  No CUDA graphs.
 *   tcqr_vgroup_create: nranks in [1, 8]; slot_bytes >= the largest collective message (e.g.
 *     4 n^2 for an n-column factor: the top R12 block is n^2/4 floats).  Allocates 2 * nranks
 *     device slots on the current device.  Returns NULL on failure.
 *   tcqr_init_virtual: rank in [0, nranks); the other arguments as tcqr_init.  Errors -3 group,
 *     -4 rank, or tcqr_init's.  A rank whose call fails aborts the group: its peers' pending
 *     collectives return TCQR_ERR_NCCL instead of waiting (host barrier timeout 120 s).
 *   tcqr_vgroup_destroy: after every rank has called tcqr_finalize.
 * ------------------------------------------------------------------------------------------- */
void* tcqr_vgroup_create(int nranks, size_t slot_bytes);
int tcqr_init_virtual(int device, void* cuda_stream, void* group, int rank);
int tcqr_vgroup_destroy(void* group);

/* Library build/version string. */
const char* tcqr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TCQR_H_ */
