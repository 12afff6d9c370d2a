// kernels.h -- internal host-side launch wrappers of the hot-path kernels (not part of the ABI).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tcqr {

constexpr int kModeTN = 0;
constexpr int kModeNN = 1;

// ---- K3 / K4 (k_gemm_tc.cu) ----
// Alg. 2 line 8 finalize targets (R block, scaled FP16 copy, column scales): when given to
// tc_gemm_tn, the split-K reduction is fused with the finalize (no separate C pass).
struct R12Finalize {
  float* Rblk;
  long long ldr;
  __half* R12h;
  long long ldh2;
  float* inv_s2;
  int scaling;
};
cudaError_t tc_gemm_tn(int m, int h, int w2, const __half* A1h, long long lda1, const __half* A2h,
                       long long lda2, float* C, long long ldc, const float* col_mult, float* P,
                       long long p_cap, int num_sms, cudaStream_t st,
                       const R12Finalize* fin = nullptr);
cudaError_t r12_splitk_finalize(int h, int w2, const float* P, int splits, long long pstride,
                                long long ldp, const float* col_mult, float* Rblk, long long ldr,
                                __half* R12h, long long ldh2, float* inv_s2, int scaling,
                                cudaStream_t st);
cudaError_t tc_gemm_nn_update(int m, int h, int w2, const __half* Qh, long long ldq,
                              const __half* Bh, long long ldb, float* C, long long ldc,
                              const float* col_mult, int num_sms, cudaStream_t st);

// ---- K1 and friends (k_cast.cu) ----
// Xh = fl16(X diag(s)); inv_s[j] = 1/s_j; status: atomicMin(1-based first non-finite column).
// m <= 65536 with aligned pointers: one thread-block cluster per column (cmax unused).  Taller:
// cmax = w uints of scratch for the split-row column max (may be null -> one CTA per column).
// src non-null (copy-cast): the columns are read from src (ld lds), the factorization's input,
// and their FP32 copy written to X in the same pass (first touch of those columns).
cudaError_t cast_scale(int m, int w, const float* X, long long ldx, __half* Xh, long long ldh,
                       float* inv_s, int scaling, int* status, int col_base, unsigned int* cmax,
                       cudaStream_t st, const float* src = nullptr, long long lds = 0);
// NEXT-4 FP16 split: Xl = fl16(X diag(s) - Xh) (inv_s null: s = 1); dst += a + b.
cudaError_t cast_lo(int m, int w, const float* X, long long ldx, const __half* Xh, long long ldh,
                    const float* inv_s, __half* Xl, long long ldl, cudaStream_t st);
cudaError_t add3(long long n, float* dst, const float* a, const float* b, cudaStream_t st);
// R12 finalize: T (h x w2, ldt) -> R block (ldr) and fl16(R12 diag(s')) (ldh2), inv_s2.
cudaError_t r12_finalize(int h, int w2, const float* T, long long ldt, float* Rblk, long long ldr,
                         __half* R12h, long long ldh2, float* inv_s2, int scaling, cudaStream_t st);
// Copy A -> Q (ld m) and flag the first non-finite column in status.
cudaError_t copy_validate(int m, int n, const float* A, long long lda, float* Q, long long ldq,
                          int* status, cudaStream_t st, int col0 = 0);
// Copy an h x w block (ld src / dst).
cudaError_t copy_block(int h, int w, const float* S, long long lds, float* D, long long ldd,
                       cudaStream_t st);
// C = A * B for upper-triangular A, B (n x n, FP32, column-major); C upper triangular.
// X <- I - X (n x n).
cudaError_t eye_minus(int n, float* X, long long ldx, cudaStream_t st);
cudaError_t trmm_upper(int n, const float* A, long long lda, const float* B, long long ldb,
                       float* C, long long ldc, cudaStream_t st);
// Zero the strictly lower triangle of an n x n matrix (ld).
cudaError_t zero_lower(int n, float* R, long long ldr, cudaStream_t st);

// ---- K2 panel (k_panel.cu) ----
// One CAQR level: MGS on each br-row block of X (rows x w), local Q in place, R_b -> stack rows
// [b*w, (b+1)*w) of S (lds), or (nb == 1) -> Rout (ldr).  top: zero norms are errors.
cudaError_t panel_mgs_level(int rows, int w, float* X, long long ldx, int br, int nb, float* S,
                            long long lds, float* Rout, long long ldr, int top, int* status,
                            int col0, cudaStream_t st);
// Step 4 of Eq. (6): X_b <- X_b * S[b*w:(b+1)*w, :].
cudaError_t panel_apply(int rows, int w, float* X, long long ldx, int br, int nb, const float* S,
                        long long lds, cudaStream_t st);
int panel_num_blocks(int rows, int br, int w);
// Fused single-launch Eq. (6) panel (cooperative); cudaErrorNotSupported -> use the levels above.
cudaError_t panel_fused(int m, int w, float* X, long long ldx, __half* Xh, long long ldh, int br,
                        float* Rout, long long ldr, int root_is_global, int* status, int col0,
                        float* ws, long long ws_cap, int* iws, long long iws_cap, int num_sms,
                        cudaStream_t st);
int fused_panel_capacity(int num_sms);
// Pipelined single-level panel (root runs one MGS step behind the row blocks); Rb, S: NaN-filled
// scratch (32*32*32 floats each), left NaN-filled.  cudaErrorNotSupported -> panel_fused.
cudaError_t panel_pipe(int m, int w, float* X, long long ldx, __half* Xh, long long ldh, int br,
                       float* Rout, long long ldr, int root_is_global, int* status, int col0,
                       float* Rb, float* S, int num_sms, cudaStream_t st);
int fused_panel_smem_bytes();
int fused_panel_max_rows();
extern unsigned long long* g_panel_dbg;
extern unsigned long long* g_proj_dbg;  // debug: phase timestamps of the FP32 projection  // debug: phase timestamps of the fused panel

// ---- K2L whole-leaf kernel (k_leaf.cu) ----
// The leaf columns [0, wl) of X (m rows, ldx; wl <= 128) factored in one cooperative launch:
// Q in place (and its FP16 shadow into Xh when non-null), R(i, j) of the leaf at R[i + j ldr].
// tg: leaf_tag_words() 64-bit words, zeroed together with tag_seq[0] = 0 (the host's count of the
// tagged reductions used so far, advanced by each launch).  num_sms: the launch's SM budget.
// cudaErrorNotSupported when the blocks do not fit the co-resident grid.
size_t leaf_tag_words();
extern unsigned long long* g_leaf_dbg;  // debug: CTA-0 phase timestamps of the leaf kernel
extern unsigned long long* g_leaf_dbg_multi;  // debug: 128 launches x 128 phase slots
extern unsigned g_leaf_dbg_idx;
extern unsigned long long* g_leaf_trace;  // debug: per-launch (start, end) of every leaf launch
cudaError_t leaf_fused(int m, int wl, float* X, long long ldx, __half* Xh, long long ldh, float* R,
                       long long ldr, int col0, int* status, unsigned long long* tg,
                       unsigned* tag_seq, int num_sms, cudaStream_t st);

// Replicated leaf across ranks: pack the rank's m x w rows into an mpad x w block (ld mpad, zero
// rows past m); unpack rows of a factored panel (ld lds) into X and its FP16 shadow Xh (nullable).
cudaError_t pack_rows(int m, int w, const float* X, long long ldx, int mpad, float* dst,
                      cudaStream_t st);
cudaError_t unpack_rows(int m, int w, const float* src, long long lds, float* X, long long ldx,
                        __half* Xh, long long ldh, cudaStream_t st);

// X (m x w, ldx; w <= 128) <- X S (S w x w, lds; FP32), FP16 shadow of the result into Xh if
// non-null: Eq. (6) step 4 for the per-leaf TSQR across ranks.
cudaError_t apply_right(int m, int w, float* X, long long ldx, const float* S, long long lds,
                        __half* Xh, long long ldh, cudaStream_t st);

// ---- K2b FP32 intra-leaf products (k_f32.cu) ----
// T (h x w2, ld h) = Q1' A2 over m rows (deterministic split-K with partials in P).
cudaError_t f32_tn(int m, int h, int w2, const float* Q1, long long ldq, const float* A2,
                   long long lda, float* T, float* P, long long p_cap, int num_sms,
                   cudaStream_t st);
// Fused (one cooperative launch): T = R12 = Q1' A2, R block <- T, A2 -= Q1 T.  bar: two zeroed
// ints.  cudaErrorNotSupported -> use f32_tn / f32_nn_update.
cudaError_t f32_project(int m, int h, int w2, const float* Q1, long long ldq, float* A2,
                        long long lda, float* Rblk, long long ldr, float* T, float* P,
                        long long p_cap, int* bar, int num_sms, cudaStream_t st);
// A2 (m x w2) -= Q1 (m x h) T (h x w2, ld h).
cudaError_t f32_nn_update(int m, int h, int w2, const float* Q1, long long ldq, const float* T,
                          float* A2, long long lda, cudaStream_t st);

// ---- CGLS (k_cgls.cu) ----
struct CglsDev;  // device state, see k_cgls.cu
cudaError_t trinv_f64(int n, const float* R, long long ldr, double* M, long long ldm, double* work,
                      int num_sms, cudaStream_t st);
cudaError_t gemv_f32_n(int m, int n, const float* A, long long lda, const double* v, double* y,
                       double* part, long long part_cap, cudaStream_t st);
// part: cg_gemv_t_part_count(m, n) doubles of scratch
cudaError_t gemv_f32_t(int m, int n, const float* A, long long lda, const double* v, double* y,
                       double* part, cudaStream_t st);

}  // namespace tcqr
