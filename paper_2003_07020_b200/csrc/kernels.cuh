// kernels.cuh -- declarations of the sm_100a kernels and their host launchers.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace fpc {

// Twiddle tables: for every N = 2^k (k <= kMaxLogTw) the table tw_N[t] = e^{-2 pi i t/N},
// t < N, lives at tw_base + N.
constexpr int kMaxLogTw = 17;

// Kernel-launch counter (fpc_kernel_launches): every launch site of the library calls it once per
// kernel it enqueues (a launcher may enqueue several, e.g. the 2D matvec's row and column passes).
void note_launch();

// Shared-memory carveout for a kernel: the smallest supported shared-memory capacity (sm_100: 0, 8,
// 16, 32, 64, 100, 132, 164, 196, 228 KB per SM) that still holds the CTAs per SM the kernel's
// register budget allows (threads: <=64 -> 8, <=128 -> 4, <=256 -> 2, else 1), so the rest of the 256 KB
// L1/shared array stays L1 for the twiddle and eigenvalue tables.  FPC_CARVEOUT=max restores
// the maximum shared-memory carveout.
int carveout_pct(size_t dyn_smem, int threads);

// ---- 1D all-at-once matvec (all_at_once.hpp:33-55 + toeplitz.hpp:41-57) --------------------
// y_k = C-stencil(v)_k + IFFT(eig' .* FFT(pad(v_k)))  with eig' = -dt*eig/(2L) pre-folded.
// koff = global time level of v's first block (time-sharded callers: the two previous blocks
// must sit right before v in memory when koff > 0).
cudaError_t launch_matvec_1d(const double* v, double* y, int n_space, int n_time, int log_m,
                             const double* eig_scaled, const double2* tw_base, cudaStream_t st,
                             int koff = 0);

// M = 8192 / 16384 (Ns up to 8191 / 16383) on a 2-CTA cluster (kernels_mv.cu).  eig_scaled also
// holds, at double offset eigq_offset(M), the per-rank table {eig'[kap], eig'[M - kap]} (kap = 2t+2
// for rank 0, 2t+1 for rank 1, t < M/4) the kernel's spectral product reads contiguously.
__host__ __device__ constexpr int eigq_offset(int m) { return (m + 1 + 1) & ~1; }
cudaError_t launch_matvec_split(const double* v, double* y, int n_space, int n_time, int log_m, int koff,
                                const double* eig_scaled, const double2* tw_base, cudaStream_t st);

// Ns + 1 = 32768 .. 65536 (kernels_large.cu): clusters of C = L/8192 CTAs (8, 16)
cudaError_t launch_matvec_large(const double* v, double* y, int n_space, int n_time, int log_m, int koff,
                                const double* eig_scaled, const double2* tw_base, cudaStream_t st);

// ---- preconditioner apply, reference ordering (alpha_circulant.hpp:137-199) ---------------
// K2: Z[n][p] = sum_k s_in*scale_fwd[k]*v[k][p] e^{+2 pi i kn/Nt}, n = 0..Nt/2 (half spectrum).
cudaError_t launch_time_fwd(const double* v, double2* Z, int n_space, int n_time,
                            const double* scale_fwd, double s_in, const double2* tw_base,
                            cudaStream_t st);
// K4: z[k][p] = Re( scale_bwd[k]/Nt * sum_n Z_n e^{-2 pi i kn/Nt} ), Z_{Nt-n} = conj(Z_n).
cudaError_t launch_time_inv(const double2* Z, double* z, int n_space, int n_time,
                            const double* scale_bwd, const double2* tw_base, cudaStream_t st);
// K2 / K4 for n_time = 128..512 on persistent CTAs fed by TMA (kernels_time_tma.cu): used when the
// grid has at least two waves of column tiles and the input is 16-byte aligned; FPC_TIME_TMA=0
// keeps the register-staged kernels (A/B).
bool time_tma_supported(int n_space, int n_time, const void* in, bool inverse);
// n_time = 1024 on warp-owned 512-point transforms, one column per warp (kernels_time_warp.cu)
bool time_warp_supported(int n_space, int n_time);
cudaError_t launch_time_fwd_warp(const double* v, double2* Z, int n_space, int n_time, const double* scale_fwd,
                                 double s_in, const double2* tw_base, cudaStream_t st);
cudaError_t launch_time_inv_warp(const double2* Z, double* z, int n_space, int n_time, const double* scale_bwd,
                                 const double2* tw_base, cudaStream_t st);
cudaError_t launch_time_fwd_tma(const double* v, double2* Z, int n_space, int n_time, const double* scale_fwd,
                                double s_in, const double2* tw_base, cudaStream_t st);
cudaError_t launch_time_inv_tma(const double2* Z, double* z, int n_space, int n_time, const double* scale_bwd,
                                const double2* tw_base, cudaStream_t st);
// InnerSweep::full (kernels_full.cu): mirror-fill rows Nt/2+1..Nt-1 of a full [Nt][ns] spectrum,
// and the complex inverse time FFT with the imaginary-residue partials (partial[blk*2 + {0,1}] =
// {sum Im^2, sum |.|^2}, dots_grid() CTAs).
cudaError_t launch_mirror_fill(double2* Z, int n_space, int n_time, cudaStream_t st);
cudaError_t launch_time_inv_full(const double2* Z, double* z, int n_space, int n_time,
                                 const double* scale_bwd, const double2* tw_base, double* partial,
                                 cudaStream_t st);
// K3 (1D): for each retained n: Z_n <- DST( DST(Z_n) ./ (lambda_n - dt*sigma) )
// (forward = true: .* instead of ./, the apply_forward action tau.hpp:132-136).
cudaError_t launch_tau_solve_1d(double2* Z, int n_space, int n_rows, const double2* lambda,
                                const double* sigma, double dt, const double2* tw_base,
                                cudaStream_t st, bool forward = false);

// Ns + 1 = 16384 .. 65536 (kernels_large.cu): DST-I via the odd extension on clusters of 2N/8192 CTAs
cudaError_t launch_tau_large(double2* Z, int n_space, int n_rows, const double2* lambda, const double* sigma,
                             double dt, const double2* tw_base, cudaStream_t st, bool forward);

// Toeplitz along nrows contiguous rows of length len (row r at v + r*len, time level r / rpt) +
// BDF2 stencil with stride sstride: 1D (rpt=1, sstride=len) and the 2D y-direction pass.
cudaError_t launch_matvec_rows(const double* v, double* y, int len, int nrows, int rpt,
                               int sstride, int log_m, const double* eig_scaled,
                               const double2* tw_base, cudaStream_t st, int koff = 0);
// the same on warp-owned register FFTs (kernels_warp.cu) for log_m = 8; cudaErrorNotSupported
// otherwise.  Used by launch_matvec_rows unless the environment sets FPC_WARP=0 (A/B).
cudaError_t launch_matvec_rows_warp(const double* v, double* y, int len, int nrows, int rpt, int sstride,
                                    int log_m, const double* eig_scaled, const double2* tw_base,
                                    cudaStream_t st, int koff);
bool warp_kernels_enabled();
// the same for M = 1024 (rows / columns of 513..1023 points: config 3's n = 1023) on one warp per
// transform, 32 lanes x 32 registers (kernels_warp32.cu).  FPC_W32=0 keeps the CTA-level kernels (A/B).
bool warp32_kernels_enabled();
int warp32_min_rows();
cudaError_t launch_matvec_rows_w32(const double* v, double* y, int len, int nrows, int rpt, int sstride,
                                   const double* eig_scaled, const double2* tw_base, cudaStream_t st, int koff);
cudaError_t launch_dst_rows_w32(double2* Z, int n, int n_rows, const double2* lambda, const double* sigma,
                                double dt, const double2* tw_base, cudaStream_t st, int mode);
cudaError_t launch_tau_cols_w32(double2* Z, int n, int n_planes, const double2* lambda, const double* sigma,
                                double dt, const double2* tw_base, cudaStream_t st, bool forward);
cudaError_t launch_matvec_cols_w32(const double* v, double* y, int n, int n_time, const double* eig_x,
                                   const double2* tw_base, cudaStream_t st);
// the 2D tau solve's column pass (DST, shift, DST along ix) on warp-owned transforms for n = 255
cudaError_t launch_tau_cols_warp(double2* Z, int n, int n_planes, const double2* lambda, const double* sigma,
                                 double dt, const double2* tw_base, cudaStream_t st, bool forward);
// the 2D matvec's x-direction column pass on warp-owned transforms for log_m = 8 (n <= 255)
cudaError_t launch_matvec_cols_warp(const double* v, double* y, int n, int n_time, int log_m, const double* eig_x,
                                    const double2* tw_base, cudaStream_t st);
// DST rows of n = 255 on warp-owned transforms (kernels_warp.cu): mode 0 = in-place DST of each row,
// 1 / 2 = DST, divide / multiply by lambda_row - dt sigma, DST (the 1D tau solve / forward action).
// cudaErrorNotSupported for other n.
cudaError_t launch_dst_rows_warp(double2* Z, int n, int n_rows, const double2* lambda, const double* sigma,
                                 double dt, const double2* tw_base, cudaStream_t st, int mode);
// in-place orthonormal DST-I of n_rows contiguous complex rows of length n (n + 1 = 2^k)
cudaError_t launch_dst_rows(double2* Z, int n, int n_rows, const double2* tw_base, cudaStream_t st);

// ---- 2D (jacobian.hpp:77-94, tau.hpp:79-96) -----------------------------------------------
cudaError_t launch_matvec_2d(const double* v, double* y, int n, int n_time, int log_m,
                             const double* eig_y_scaled, const double* eig_x_scaled,
                             const double2* tw_base, cudaStream_t st, int koff = 0);
// scratch (optional, n_rows * n * n complex): with it the n = 255 solve runs without strided loads
// (two row passes with transposed stores through scratch, kernels_warp.cu k_dst_rows_T)
cudaError_t launch_tau_solve_2d(double2* Z, int n, int n_rows, const double2* lambda,
                                const double* sigma, double dt, const double2* tw_base,
                                cudaStream_t st, bool forward = false, double2* scratch = nullptr);
cudaError_t launch_dst_rows_T(const double2* in, double2* out, int n, int n_planes, const double2* lambda,
                              const double* sigma, double dt, const double2* tw_base, cudaStream_t st, int mode);

// ---- commuted ordering beyond kernels_commuted.cu's 1D n_space + 1 <= 8192 -------------------
// time-level pairs as complex levels (kernels_2d.cu), one DST per complex row for n_space + 1 =
// 16384..65536 (kernels_large.cu), one DST along the columns of n_planes 2D planes (kernels_2d.cu)
cudaError_t launch_pack_pairs(const double* v, double2* U, int ns, int n_levels, double s, cudaStream_t st);
cudaError_t launch_unpack_pairs(const double2* U, double* v, int ns, int n_levels, cudaStream_t st);
cudaError_t launch_dst_large(double2* Z, int n_space, int n_rows, const double2* tw_base, cudaStream_t st);
cudaError_t launch_dst_cols_2d(double2* Z, int n, int n_planes, const double2* tw_base, cudaStream_t st);

// ---- generic sizes (kernels_generic.cu): Bluestein transforms along a strided batch ---------
// sequence s (s < count) element j sits at data + (s / inner) * outer_stride + (s % inner) *
// inner_stride + j * es; chirp / bhat as fft.hpp:71-89 (host-built); len <= 4096.
// (sign = the transform's kernel sign; a power-of-two len runs the plain transform, no chirp)
cudaError_t launch_bluestein(double2* data, int len, long long count, long long inner, long long outer_stride,
                             long long inner_stride, long long es, const double2* chirp, const double2* bhat,
                             const double2* tw_base, cudaStream_t st, int sign);
cudaError_t launch_gen_time_in(const double* v, double2* U, int ns, int nt, const double* sf, double s_in,
                               cudaStream_t st);
cudaError_t launch_gen_time_out(const double2* U, double* z, int ns, int nt, const double* sb, cudaStream_t st);
// + the imaginary-residue partials (dots_grid() blocks x {Im^2, |.|^2}) for InnerSweep::full
cudaError_t launch_gen_time_out_guard(const double2* U, double* z, int ns, int nt, const double* sb, double* partial,
                                      cudaStream_t st);
cudaError_t launch_gen_mirror(double2* U, int nt, int ns, int h, cudaStream_t st);
// DST-I (odd extension, length-2(n+1) Bluestein transform, extraction) of `count` strided
// sequences of n complex values in place; mode 1 / 2 divides / multiplies the DST output by
// lambda_f - dt sigma (f = s / per_freq, sigma at the element's offset minus f * plane).
cudaError_t launch_gen_dst(double2* U, double2* D, int n, long long count, long long inner, long long outer_stride,
                           long long inner_stride, long long es, const double2* chirp, const double2* bhat,
                           const double2* tw_base, int mode, long long per_freq, long long plane, const double2* lam,
                           const double* sigma, double dt, cudaStream_t st);

// ---- Krylov vector kernels (krylov.hpp:52-62, 116-131, 166-167, 180-182) -------------------
struct VecSet {
  const double* v[8];
  double s[8];
};
// partial[blk*stride + i] = s_i * sum v_i .* w  (i < nv), partial[blk*stride + nv] = sum w.*w
// when with_norm.  Deterministic: fixed grid, fixed in-block tree.
int dots_grid();
cudaError_t launch_dots(const VecSet& vs, int nv, const double* w, size_t n, double* partial,
                        int stride, int col0, bool with_norm, cudaStream_t st);
// out[i] = sum_b partial[b*stride + i], i < count (fixed order); optional accumulate into out.
cudaError_t launch_reduce(const double* partial, int stride, int count, double* out,
                          bool accumulate, cudaStream_t st);
// w <- w - sum_i c_i v_i with c_i = coef[i]*s_i (coef on device); partial norm of the result.
cudaError_t launch_update(const double* const* vptr, const double* scales, const double* coef,
                          int nv, double* w, size_t n, double* partial, cudaStream_t st);
// fused: w <- w - sum_i coef_i s_i v_i; partial[blk*stride + i] = s_i <v_i, w_new> (i < nv) and
// partial[blk*stride + nv] = ||w_new||^2.  nv <= kMaxFused.
constexpr int kMaxFused = 24;
struct VecSetN {
  const double* v[kMaxFused];
  double s[kMaxFused];
};
cudaError_t launch_update_dots(const VecSetN& vs, int nv, const double* coef, double* w, size_t n,
                               double* partial, int stride, cudaStream_t st);
// u = sum_i c_i * s_i * v_i (c on device)
cudaError_t launch_lincomb(const double* const* vptr, const double* scales, const double* coef,
                           int nv, double* u, size_t n, cudaStream_t st);
// partial = sum (b - y)^2 ; partial over blocks (reduce with launch_reduce)
cudaError_t launch_resid_norm(const double* b, const double* y, size_t n, double* partial,
                              cudaStream_t st);
// y = a*x + y
cudaError_t launch_axpy(double a, const double* x, double* y, size_t n, cudaStream_t st);
// y = b - y
cudaError_t launch_rsub(const double* b, double* y, size_t n, cudaStream_t st);

// ---- delayed re-orthogonalisation Gram-Schmidt (api.cu gmres_inner_lagged) ----------------
constexpr int kDots2B = 128;  // partial column offset of the b_i = <v_i, W> block
constexpr int kDots2X = 256;  // partial columns of <U,W>, <U,U>, <W,W>
struct VecSet16 {
  const double* v[16];
  double s[16];
};
// partial[blk*stride + col0 + i] = s_i <v_i, U>, [.. + kDots2B + col0 + i] = s_i <v_i, W> (i < nv <= 16),
// extra: [.. + kDots2X + 0..2] = <U,W>, <U,U>, <W,W>
cudaError_t launch_dots2(const VecSet16& vs, int nv, const double* U, const double* W, size_t n,
                         double* partial, int stride, int col0, bool extra, cudaStream_t st);
// out[c] for the used columns of a dots2 reduction only (c = 0..nab-1, kDots2B + 0..nab-1,
// kDots2X + 0..2), same per-column arithmetic as launch_reduce
cudaError_t launch_reduce_dots2(const double* partial, int stride, int nab, double* out, cudaStream_t st);
constexpr int kMaxUpd2 = 24;
struct Update2Args {
  const double* v[kMaxUpd2];
  double ca[kMaxUpd2];
  double cd[kMaxUpd2];
  double cu, cw;
};
// U <- U - sum ca_i v_i; W <- (first ? cw W + cu U_old : W) + sum cd_i v_i; norm: partial = ||W||^2
// keep_u: U is read (first group: the cu term) but not updated or written
cudaError_t launch_update2(const Update2Args& a, int nv, bool first, bool norm, double* U, double* W,
                           size_t n, double* partial, cudaStream_t st, bool keep_u = false);

// ---- commuted preconditioner ordering (kernels_commuted.cu), 1D --------------
// out = S v per time level, levels (k, k + Nt/2) paired in one complex row; scale s_in
cudaError_t launch_dst_pairs(const double* v, double* out, int n_space, int n_time, double s_in,
                             const double2* tw_base, cudaStream_t st);
// per spatial column p: z = D^{-1} F^* diag(1/(lambda_n - dt sigma_p)) F D (s_in u)  (forward: multiply)
cudaError_t launch_time_solve(const double* u, double* z, int n_space, int n_time, const double* scale_fwd,
                              const double* scale_bwd, double s_in, const double2* lambda, const double* sigma,
                              double dt, const double2* tw_base, cudaStream_t st, bool forward);

// ---- time FFTs on 2-CTA clusters split by time parity (kernels_tsplit.cu), Nt = 1024 / 2048:
// the launchers above dispatch to these when time_split_supported(n_time)
bool time_split_supported(int n_time);
cudaError_t launch_time_fwd_split(const double* v, double2* Z, int n_space, int n_time, const double* scale_fwd,
                                  double s_in, const double2* tw_base, cudaStream_t st);
cudaError_t launch_time_inv_split(const double2* Z, double* z, int n_space, int n_time, const double* scale_bwd,
                                  const double2* tw_base, cudaStream_t st);
cudaError_t launch_time_solve_split(const double* u, double* z, int n_space, int n_time, const double* scale_fwd,
                                    const double* scale_bwd, double s_in, const double2* lambda,
                                    const double* sigma, double dt, const double2* tw_base, cudaStream_t st,
                                    bool forward);

// ---- BiCGSTAB vector kernels (krylov.hpp:204-280) -------------------------------------------
// p = r (first) or r + beta (p - omega v)
cudaError_t launch_bicg_p(const double* r, const double* v, double* p, double beta, double omega,
                          size_t n, bool first, cudaStream_t st);
// alpha = rho_denom[0]/rho_denom[1]; r <- r - alpha v (= s); rt <- rt - alpha q (= s_true);
// partial[blk] = ||s_true||^2
cudaError_t launch_bicg_s(double* r, double* rt, const double* v, const double* q,
                          const double* rho_denom, size_t n, double* partial, cudaStream_t st);
// x += alpha p + omega s; r <- s - omega t; rt <- s_true - omega t_orig;
// partial[blk*2] = ||rt||^2, partial[blk*2+1] = <rhat, r>
cudaError_t launch_bicg_x(double* x, const double* p, double* r, const double* t, double* rt,
                          const double* to, const double* rhat, double alpha, double omega,
                          size_t n, double* partial, cudaStream_t st);

// kernels_p2p.cu: one exchange of the sharded PC apply as peer stores (destinations by kernel param)
constexpr int kP2PMaxRanks = 8;
struct P2PScatter {
  double* dst[kP2PMaxRanks];  // receive buffer of each rank (peer-mapped, or local for the own rank)
  int off[kP2PMaxRanks];      // partition of the split dimension: rank d owns [off[d], off[d+1])
  int stride[kP2PMaxRanks];   // row stride (elements) of rank d's receive matrix
};
cudaError_t launch_p2p_scatter(const double* src, int rows, int cols, int es, bool split_cols, const P2PScatter& a,
                               int nranks, int row_base, int col_base, cudaStream_t st);

}  // namespace fpc
