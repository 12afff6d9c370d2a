// cgls_state.h -- device-resident CGLS state (Alg. 5 scalars + the R-A11 stop bookkeeping).
#pragma once
#include <cuda_runtime.h>

namespace tcqr {

struct CgState {
  double gamma;   // ||s_k||^2 (Alg. 5 line 10 / 22)
  double delta;   // ||q_k||^2 (line 14)
  double s0;      // ||s_0|| of this pass
  double sref;    // ||s_0|| of pass 1 (stagnation floor reference, R-A11)
  double best;    // smallest ||s_k|| seen this pass
  double tol;     // stop when ||s_k|| / ||s_0|| <= tol
  double floor;   // stagnation floor (relative to sref)
  int k;          // iterations done this pass
  int since;      // iterations since the last new best
  int window;     // stagnation window W
  int maxit;
  int done;       // 1 once stopped: every CGLS kernel then returns immediately
  int reason;     // 0 tol, 1 stagnation, 2 maxit, 3 zero rhs
  int hist_cap;
  int pad;
};

int cg_gemv_n_chunks(int n);
int cg_tri_chunks(int n);
cudaError_t cg_launch_tri_n(int n, const double* M, long long ldm, const double* p, double* t,
                            double* part, const int* done, cudaStream_t st);
cudaError_t cg_launch_tri_t(int n, const double* M, long long ldm, const double* v, double* s,
                            const int* done, cudaStream_t st);
// FP32 copy of the preconditioner M = R^-1 (reading R-A13): same products, FP64 accumulation.
cudaError_t cg_launch_tri_n(int n, const float* M, long long ldm, const double* p, double* t,
                            double* part, const int* done, cudaStream_t st);
// s = M' v for the FP32 M (part: cg_tri_t_part_count(n) doubles)
int cg_tri_t_part_count(int n);
cudaError_t cg_launch_tri_t(int n, const float* M, long long ldm, const double* v, double* s,
                            double* part, const int* done, cudaStream_t st);
cudaError_t cg_launch_m_to_f32(int n, const double* M, long long ldm, float* M32, cudaStream_t st);
cudaError_t cg_launch_a_n(int m, int n, const float* A, long long lda, const double* t, double* q,
                          double* part, double* dpart, const int* done, cudaStream_t st);
// v = A' r (part: cg_gemv_t_part_count(m, n) doubles).  With q and cst: v = A' (r - alpha q),
// alpha = cst->gamma / cst->delta, and r - alpha q is written to r_out (Alg. 5 line 17 fused).
int cg_gemv_t_part_count(int m, int n);
cudaError_t cg_launch_a_t(int m, int n, const float* A, long long lda, const double* r, double* v,
                          double* part, const int* done, cudaStream_t st,
                          const double* q = nullptr, const CgState* cst = nullptr,
                          double* r_out = nullptr);
// x += alpha t (alpha = gamma / delta), Alg. 5 line 16.
cudaError_t cg_launch_update_x(int n, CgState* s, double* x, const double* t, cudaStream_t st);
cudaError_t cg_launch_sum_parts(int np, const double* parts, double* out, const int* done,
                                cudaStream_t st);
cudaError_t cg_launch_update_xr(int m, int n, CgState* s, double* x, const double* t, double* r,
                                const double* q, cudaStream_t st);
cudaError_t cg_launch_init(int n, CgState* s, const double* sv, double* p, double* x,
                           double* xbest, cudaStream_t st);
cudaError_t cg_launch_finish(int n, CgState* s, const double* sv, double* p, double* x,
                             double* xbest, double* hist, cudaStream_t st);
cudaError_t cg_launch_residual(int m, const double* b, const double* q, double* r,
                               cudaStream_t st);
cudaError_t cg_launch_axpy(int n, double a, const double* x, double* y, cudaStream_t st);

}  // namespace tcqr
