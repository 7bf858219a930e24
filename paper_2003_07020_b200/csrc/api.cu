// api.cu -- the C-ABI (include/fracpint_b200.h): contexts, problems (operator setup on the host,
// device-resident spectra), preconditioner plans and the device-resident GMRES driver.
//
// Host-side setup restates the reference's one-off constructions (weights.hpp:21-35,
// toeplitz.hpp:23-35, tau.hpp:40-73, alpha_circulant.hpp:71-126) in double precision on the CPU;
// everything per-iteration runs on the GPU (kernels_1d.cu, kernels_2d.cu, kernels_krylov.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <mutex>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/fracpint_b200.h"
#include "kernels.cuh"

namespace {

thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct CudaFail {
  cudaError_t err;
  const char* what;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail{e, what};
}
bool debug_sync() {
  static const bool on = [] {
    const char* e = std::getenv("FPC_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}
inline void ckl(cudaError_t e, const char* what) {  // kernel launch (counted by fpc::note_launch)
  ck(e, what);
  if (debug_sync()) ck(cudaDeviceSynchronize(), what);
}

// Live per-kernel timing (fpc_profile_*): CUDA events recorded on the launching stream around
// every launch while enabled; resolved after the caller synchronizes.
struct Profiler {
  bool on = false;
  struct Pending {
    cudaEvent_t a, b;
    int cat;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  std::vector<std::string> names;
  std::vector<double> ms;
  std::vector<long long> count;
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  int cat(const char* name) {
    for (size_t i = 0; i < names.size(); ++i)
      if (names[i] == name) return int(i);
    names.emplace_back(name);
    ms.push_back(0.0);
    count.push_back(0);
    return int(names.size()) - 1;
  }
  void resolve() {
    for (auto& p : pending) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
        ms[size_t(p.cat)] += t;
        count[size_t(p.cat)] += 1;
      }
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
};
Profiler g_prof;

struct ProfScope {
  cudaStream_t st;
  int cat = -1;
  cudaEvent_t a{};
  ProfScope(const char* name, cudaStream_t s) : st(s) {
    if (!g_prof.on) return;
    cat = g_prof.cat(name);
    a = g_prof.get();
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (cat < 0) return;
    cudaEvent_t b = g_prof.get();
    cudaEventRecord(b, st);
    g_prof.pending.push_back({a, b, cat});
  }
};
#define LAUNCH(name, stream, call)   \
  do {                               \
    ProfScope ps_(name, stream);     \
    ckl((call), name);               \
  } while (0)

struct InvalidArg {
  std::string msg;
};
struct RuntimeErr {
  std::string msg;
};
struct Unsupported {
  std::string msg;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FPC_OK;
  } catch (const InvalidArg& e) {
    return set_err(FPC_INVALID_ARGUMENT, e.msg);
  } catch (const RuntimeErr& e) {
    return set_err(FPC_RUNTIME_ERROR, e.msg);
  } catch (const Unsupported& e) {
    return set_err(FPC_UNSUPPORTED, e.msg);
  } catch (const CudaFail& e) {
    return set_err(FPC_CUDA_ERROR, std::string(e.what) + ": " + cudaGetErrorString(e.err));
  } catch (const std::bad_alloc&) {
    return set_err(FPC_RUNTIME_ERROR, "host allocation failed");
  } catch (const std::exception& e) {
    return set_err(FPC_RUNTIME_ERROR, e.what());
  }
}

using cplx = std::complex<double>;
constexpr double kPi = 3.14159265358979323846264338327950288;

int ilog2_exact(size_t n) {
  int l = 0;
  while ((size_t(1) << l) < n) ++l;
  return (size_t(1) << l) == n ? l : -1;
}
size_t next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// ---- host FFT for setup only (power-of-two radix-2, kernel e^{sign 2 pi i jk/n}) -----------
// The complex product as g++ contracts std::complex<double> multiplication in the reference's
// fft_pow2 butterfly (fft.hpp:62) once FMA is available (-march=native / x86-64-v3): written out,
// so the setup (circulant eigenvalues, tau spectrum) is bit-identical to the reference's whatever
// this translation unit's own contraction choices are.  At n = 65535 the tau spectrum's smallest
// eigenvalue carries ~1e-6 cancellation error in any implementation; sharing the reference's
// exact doubles keeps the large config-4 PC applies at rounding distance from the reference.
inline cplx cmul_fma(cplx a, cplx b) {
  return cplx(std::fma(a.real(), b.real(), -(a.imag() * b.imag())),
              std::fma(a.real(), b.imag(), a.imag() * b.real()));
}

void host_fft_pow2(std::vector<cplx>& x, int sign) {
  const size_t n = x.size();
  if (n <= 1) return;
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(x[i], x[j]);
  }
  const double unit = 2.0 * kPi * (sign >= 0 ? 1.0 : -1.0) / double(n);
  std::vector<cplx> tw(n / 2);
  for (size_t j = 0; j < n / 2; ++j) tw[j] = std::polar(1.0, unit * double(j));
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len >> 1, step = n / len;
    for (size_t base = 0; base < n; base += len)
      for (size_t j = 0; j < half; ++j) {
        const cplx u = x[base + j], v = cmul_fma(x[base + j + half], tw[j * step]);
        x[base + j] = u + v;
        x[base + j + half] = u - v;
      }
  }
}

// Bluestein chirp (fft.hpp:74-77) of an arbitrary length n and kernel sign
std::vector<cplx> bluestein_chirp(size_t n, int sign) {
  const double dir = sign >= 0 ? 1.0 : -1.0;
  std::vector<cplx> chirp(n);
  for (size_t m = 0; m < n; ++m) {
    const uint64_t sq = (uint64_t(m) * m) % (2 * n);
    chirp[m] = std::polar(1.0, dir * kPi * double(sq) / double(n));
  }
  return chirp;
}
// its convolution filter FFT_L^-(b), b_m = conj(chirp_|m|) circularly (fft.hpp:78-83)
std::vector<cplx> bluestein_filter(const std::vector<cplx>& chirp, size_t L) {
  const size_t n = chirp.size();
  std::vector<cplx> b(L);
  b[0] = std::conj(chirp[0]);
  for (size_t m = 1; m < n; ++m) b[m] = b[L - m] = std::conj(chirp[m]);
  host_fft_pow2(b, -1);
  return b;
}
// fft_bluestein (fft.hpp:71-89), products written as the reference's contracted ones (cmul_fma)
void host_fft_bluestein(std::vector<cplx>& x, int sign) {
  const size_t n = x.size(), L = next_pow2(2 * n - 1);
  const std::vector<cplx> chirp = bluestein_chirp(n, sign);
  std::vector<cplx> a(L);
  for (size_t j = 0; j < n; ++j) a[j] = cmul_fma(x[j], chirp[j]);
  const std::vector<cplx> b = bluestein_filter(chirp, L);
  host_fft_pow2(a, -1);
  for (size_t j = 0; j < L; ++j) a[j] = cmul_fma(a[j], b[j]);
  host_fft_pow2(a, 1);
  const double inv_L = 1.0 / double(L);
  for (size_t k = 0; k < n; ++k) x[k] = cmul_fma(chirp[k], a[k]) * inv_L;
}
// fft_inplace (fft.hpp:95-101)
void host_fft(std::vector<cplx>& x, int sign) {
  if (x.size() <= 1) return;
  if (ilog2_exact(x.size()) >= 0)
    host_fft_pow2(x, sign);
  else
    host_fft_bluestein(x, sign);
}

// orthonormal DST-I of real data (dst.hpp:21-43), any n
std::vector<double> host_dst1(const std::vector<double>& x) {
  const size_t n = x.size(), L = 2 * (n + 1);
  std::vector<cplx> v(L);
  for (size_t j = 0; j < n; ++j) {
    v[j + 1] = x[j];
    v[L - 1 - j] = -x[j];
  }
  host_fft(v, -1);
  const double scale = std::sqrt(2.0 / double(n + 1)) * 0.5;
  std::vector<double> y(n);
  for (size_t k = 0; k < n; ++k) y[k] = scale * (cplx(0.0, 1.0) * v[k + 1]).real();
  return y;
}

// weights.hpp:21-35
std::vector<double> centred_weights(double gamma, int count) {
  if (!(gamma > 1.0) || !(gamma <= 2.0))
    throw InvalidArg{"centred_weights: gamma must lie in (1, 2]"};
  if (count < 1) throw InvalidArg{"centred_weights: count must be at least 1"};
  std::vector<double> w(static_cast<size_t>(count));
  const double g0 = std::tgamma(1.0 + gamma / 2.0);
  w[0] = std::tgamma(1.0 + gamma) / (g0 * g0);
  for (int l = 0; l + 1 < count; ++l)
    w[size_t(l) + 1] = w[size_t(l)] * (double(l) - gamma / 2.0) / (double(l) + 1.0 + gamma / 2.0);
  return w;
}

// tau.hpp:40-55
std::vector<double> tau_spectrum(const std::vector<double>& a) {
  const size_t n = a.size();
  std::vector<double> c(a);
  for (size_t l = 0; l + 2 < n; ++l) c[l] -= a[l + 2];
  const std::vector<double> num = host_dst1(c);
  const double root = std::sqrt(2.0 / double(n + 1));
  std::vector<double> s(n);
  for (size_t i = 0; i < n; ++i) s[i] = num[i] / (root * std::sin(kPi * double(i + 1) / double(n + 1)));
  return s;
}

// alpha_circulant_eigenvalues (alpha_circulant.hpp:71-81)
std::vector<cplx> alpha_lambda(double a, int nt) {
  std::vector<cplx> lam(static_cast<size_t>(nt));
  const double ar = std::pow(a, 1.0 / double(nt));
  for (int i = 0; i < nt; ++i) {
    const double ang1 = 2.0 * kPi * double(i % nt) / nt;
    const double ang2 = 2.0 * kPi * double((2 * i) % nt) / nt;
    lam[size_t(i)] = 1.5 - 2.0 * ar * std::polar(1.0, ang1) + 0.5 * ar * ar * std::polar(1.0, ang2);
  }
  return lam;
}

// circulant-embedding eigenvalues (toeplitz.hpp:23-35): real parts of FFT_{-}(c), k = 0..L/2
std::vector<double> circulant_eigs(const std::vector<double>& col) {
  const size_t n = col.size(), L = next_pow2(2 * n);
  std::vector<cplx> c(L);
  c[0] = col[0];
  for (size_t j = 1; j < n; ++j) c[j] = c[L - j] = col[j];
  host_fft(c, -1);
  std::vector<double> e(L / 2 + 1);
  for (size_t k = 0; k <= L / 2; ++k) e[k] = c[k].real();
  return e;
}

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

}  // namespace

// =================================================================================== context
struct fpc_context_s {
  int refs = 1;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double2* tw = nullptr;        // twiddle tables, size-N table at tw + N
  double* partial = nullptr;    // kDotsGrid x kPartialStride
  double* dscal = nullptr;      // small device scratch (h, norms)
  double* hpin = nullptr;       // pinned host mirror of dscal
  const double** dvptr = nullptr;  // device pointer table for update/lincomb
  double* dscales = nullptr;
  cudaStream_t aux = nullptr;   // host-path result copy overlapped with the true-residual check
  cudaEvent_t aux_ev = nullptr;
  static constexpr int kPartialStride = 264;
  static constexpr int kScal = 2048;  // [1024, 1280): unit scales for x = Z y
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// =================================================================================== problem
struct fpc_problem_s {
  int refs = 1;
  std::recursive_mutex mu;  // host calls on one operator (shared staging buffers) are serialised
  fpc_context_s* ctx = nullptr;
  int two_dim = 0;
  int n = 0;   // 1D: n_space; 2D: n per dim
  int ns = 0;  // spatial unknowns
  int nt = 0;
  double dt = 0.0;
  double sx = 0.0, sy = 0.0;
  std::vector<double> colx, coly;  // 1D: colx = scaled Jacobian column; 2D: unscaled weights
  std::vector<double> sigma;       // jac.tau() spectrum (jacobian.hpp:45, 96-98)
  int log_m = 0;                   // Toeplitz packed FFT size M = L/2
  int generic = 0;                 // a size outside the power-of-two kernels: PC apply on kernels_generic.cu
  double* d_eig = nullptr;         // 1D: -dt*eig/(2L); 2D: y-axis factor
  double* d_eig_x = nullptr;       // 2D: x-axis factor
  double* d_in = nullptr;          // staging for host-pointer calls
  double* d_out = nullptr;
  size_t dim() const { return size_t(nt) * size_t(ns); }
};

struct fpc_plan_s {
  fpc_problem_s* prob = nullptr;
  std::recursive_mutex mu;  // host calls on one plan (shared spectrum scratch, GMRES workspace) are serialised
  double alpha = 0.0;
  std::vector<cplx> lambda;
  std::vector<double> scale_fwd, scale_bwd;  // alpha^{+-k/Nt} (alpha_circulant.hpp:102-106)
  int solve_count = 0;
  double min_shift_margin = 0.0;
  int n_warnings = 0;
  double* d_sf = nullptr;
  double* d_sb = nullptr;
  double2* d_lambda = nullptr;
  double* d_sigma = nullptr;
  double2* d_Z = nullptr;  // half spectrum scratch (H x ns complex)
  double2* d_ZT = nullptr; // 2D n = 255: the transposed spectrum of the tau solve's row passes (allocated on first use)
  double2* d_Zf = nullptr; // full spectrum (Nt x ns complex), InnerSweep::full only
  int sweep_mode = FPC_SWEEP_HALF;
  // generic (Bluestein) path: chirps and filter spectra of the time transforms (signs +1 / -1) and
  // of the DST odd-extension transform; the full spectrum and the odd-extension scratch
  double2 *d_ctf = nullptr, *d_btf = nullptr, *d_cti = nullptr, *d_bti = nullptr, *d_cds = nullptr, *d_bds = nullptr;
  double2 *d_U = nullptr, *d_D = nullptr;
  double2* d_P = nullptr;  // commuted ordering beyond 1D n_space + 1 <= 8192: time-level pairs as complex levels
  int ordering = FPC_ORDER_REFERENCE;  // FPC_ORDER_COMMUTED: DST-first (kernels_commuted.cu)
  // GMRES workspace (grown on demand, reused across solves)
  std::vector<double*> basis;
  std::vector<double*> zbasis;  // z_j = P^{-1} V_j kept for x = Z y (see gmres_inner)
  double* d_z = nullptr;
  double* d_u = nullptr;
  double* d_r = nullptr;
  double* d_x = nullptr;
  double* d_d = nullptr;
  double* d_b = nullptr;
};

namespace {

// Sizes of the power-of-two kernels (fast path) and of the Bluestein path (kernels_generic.cu):
// the latter covers any n_time <= 4096 and any DST length n <= 2047 (transforms of length 2(n+1)
// up to 4096, i.e. convolutions of length <= 8192 in one CTA's shared memory).
bool pow2_sizes_1d(int n_space, int n_time) {
  return ilog2_exact(size_t(n_time)) >= 0 && n_time >= 4 && n_time <= 16384 &&
         ilog2_exact(size_t(n_space) + 1) >= 0 && n_space >= 3 && n_space + 1 <= 65536;
}
bool generic_sizes(int n_dst, int n_time) {
  return n_time >= 3 && n_time <= 4096 && n_dst >= 1 && n_dst <= 2047;
}
// returns 1 when the problem takes the generic (Bluestein) PC path
int check_sizes_1d(int n_space, int n_time) {
  if (pow2_sizes_1d(n_space, n_time)) return 0;
  if (generic_sizes(n_space, n_time) && n_space <= 65535) return 1;
  throw Unsupported{"B200 path: n_time must be a power of two in [4, 16384] and n_space + 1 a power of two "
                    "<= 65536, or (any size) n_time <= 4096 and n_space <= 2047"};
}

void upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "H2D");
}

}  // namespace

namespace fpc {
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace fpc

extern "C" {

int fpc_abi_version(void) { return 2; }
const char* fpc_last_error(void) { return g_err.c_str(); }

// ---- host-side setup routines of the reference API (no device needed) ----------------------
int fpc_centred_weights(double gamma, int count, double* out) {
  if (!out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    const std::vector<double> w = centred_weights(gamma, count);
    std::copy(w.begin(), w.end(), out);
  });
}

int fpc_tau_spectrum(const double* col, int n, double* sigma) {
  if (!col || !sigma) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  if (n < 1) return set_err(FPC_INVALID_ARGUMENT, "tau_spectrum: empty first column");
  return guarded([&] {
    const std::vector<double> s = tau_spectrum(std::vector<double>(col, col + n));
    std::copy(s.begin(), s.end(), sigma);
  });
}

int fpc_circulant_eigenvalues(const double* col, int n, double* eig) {
  if (!col || !eig) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  if (n < 1) return set_err(FPC_INVALID_ARGUMENT, "SymToeplitz: empty first column");
  return guarded([&] {
    const std::vector<double> e = circulant_eigs(std::vector<double>(col, col + n));
    std::copy(e.begin(), e.end(), eig);
  });
}

int fpc_alpha_circulant_eigenvalues(double alpha, int nt, double* lambda_interleaved) {
  if (!lambda_interleaved) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  if (nt < 1) return set_err(FPC_INVALID_ARGUMENT, "alpha_circulant_eigenvalues: nt must be positive");
  return guarded([&] {
    const std::vector<cplx> l = alpha_lambda(alpha, nt);
    std::memcpy(lambda_interleaved, l.data(), l.size() * sizeof(cplx));
  });
}
unsigned long long fpc_kernel_launches(void) { return g_launches.load(); }

int fpc_profile_start(void) {
  g_prof.resolve();
  for (auto& m : g_prof.ms) m = 0.0;
  for (auto& c : g_prof.count) c = 0;
  g_prof.on = true;
  return FPC_OK;
}

int fpc_profile_stop(void) {
  cudaDeviceSynchronize();
  g_prof.resolve();
  g_prof.on = false;
  return int(g_prof.names.size());
}

int fpc_profile_entry(int i, char* name, int name_cap, double* total_ms, long long* launches) {
  if (i < 0 || size_t(i) >= g_prof.names.size()) return set_err(FPC_INVALID_ARGUMENT, "bad index");
  if (name && name_cap > 0) {
    std::strncpy(name, g_prof.names[size_t(i)].c_str(), size_t(name_cap) - 1);
    name[name_cap - 1] = 0;
  }
  if (total_ms) *total_ms = g_prof.ms[size_t(i)];
  if (launches) *launches = g_prof.count[size_t(i)];
  return FPC_OK;
}

int fpc_context_create(int device, fpc_context_t* out) {
  if (!out) return set_err(FPC_INVALID_ARGUMENT, "null output");
  return guarded([&] {
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw InvalidArg{"fpc_context_create: bad device index"};
    DeviceGuard g(device);
    auto* c = new fpc_context_s();
    c->device = device;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->own_stream = true;
    // twiddle tables tw_N[t] = polar(1, -2 pi t / N) for N = 1 .. 2^kMaxLogTw (fft.hpp:36-37)
    const size_t total = size_t(2) << fpc::kMaxLogTw;
    std::vector<double2> tw(total);
    for (int l = 0; l <= fpc::kMaxLogTw; ++l) {
      const size_t N = size_t(1) << l;
      const double unit = -2.0 * kPi / double(N);
      for (size_t t = 0; t < N; ++t) {
        const cplx w = std::polar(1.0, unit * double(t));
        tw[N + t] = make_double2(w.real(), w.imag());
      }
    }
    c->tw = dalloc<double2>(total);
    ck(cudaMemcpy(c->tw, tw.data(), total * sizeof(double2), cudaMemcpyHostToDevice), "tw upload");
    c->partial = dalloc<double>(size_t(fpc::dots_grid()) * fpc_context_s::kPartialStride);
    c->dscal = dalloc<double>(fpc_context_s::kScal);
    ck(cudaMallocHost(&c->hpin, fpc_context_s::kScal * sizeof(double)), "cudaMallocHost");
    c->dvptr = dalloc<const double*>(512);
    c->dscales = dalloc<double>(512);
    *out = c;
  });
}

// Handles are reference counted: a problem holds its context and a plan its problem, so the
// owner may destroy them in any order (e.g. Python finalizers at interpreter exit).
static void release_ctx(fpc_context_s* c) {
  if (--c->refs > 0) return;
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->stream);
  cudaFree(c->tw);
  cudaFree(c->partial);
  cudaFree(c->dscal);
  cudaFreeHost(c->hpin);
  cudaFree(c->dvptr);
  cudaFree(c->dscales);
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
    cudaEventDestroy(c->aux_ev);
  }
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int fpc_context_destroy(fpc_context_t c) {
  if (!c) return FPC_OK;
  release_ctx(c);
  return FPC_OK;
}

int fpc_context_set_stream(fpc_context_t c, void* s) {
  if (!c) return set_err(FPC_INVALID_ARGUMENT, "null context");
  DeviceGuard g(c->device);
  if (c->own_stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  c->stream = static_cast<cudaStream_t>(s);
  c->own_stream = false;
  return FPC_OK;
}

void* fpc_context_stream(fpc_context_t c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int fpc_synchronize(fpc_context_t c) {
  if (!c) return set_err(FPC_INVALID_ARGUMENT, "null context");
  return guarded([&] { ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize"); });
}

int fpc_device_alloc(fpc_context_t c, size_t bytes, void** out) {
  if (!c || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    DeviceGuard g(c->device);
    ck(cudaMalloc(out, bytes), "cudaMalloc");
  });
}

int fpc_device_free(fpc_context_t c, void* p) {
  if (!c) return set_err(FPC_INVALID_ARGUMENT, "null context");
  DeviceGuard g(c->device);
  cudaFree(p);
  return FPC_OK;
}

// ---------------------------------------------------------------------------- problems
static fpc_problem_s* new_problem(fpc_context_s* c, int nt, double dt) {
  if (nt < 3) throw InvalidArg{"TimeStencil: need at least 3 time levels"};
  if (!(dt > 0.0)) throw InvalidArg{"AllAtOnceOperator: dt must be positive"};
  auto* p = new fpc_problem_s();
  p->ctx = c;
  ++c->refs;
  p->nt = nt;
  p->dt = dt;
  return p;
}

int fpc_problem_create_1d(fpc_context_t c, double gamma, double kappa, double h, int n_space,
                          int n_time, double dt, fpc_problem_t* out) {
  if (!c || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // RieszJacobian1D ctor (jacobian.hpp:21-32)
    if (!(kappa > 0.0)) throw InvalidArg{"RieszJacobian1D: kappa must be positive"};
    if (!(h > 0.0)) throw InvalidArg{"RieszJacobian1D: h must be positive"};
    if (n_space < 1) throw InvalidArg{"RieszJacobian1D: n_space must be at least 1"};
    std::vector<double> w = centred_weights(gamma, n_space);
    if (n_time < 3) throw InvalidArg{"TimeStencil: need at least 3 time levels"};
    if (!(dt > 0.0)) throw InvalidArg{"AllAtOnceOperator: dt must be positive"};
    const int generic = check_sizes_1d(n_space, n_time);
    DeviceGuard g(c->device);
    fpc_problem_s* p = new_problem(c, n_time, dt);
    p->generic = generic;
    p->n = p->ns = n_space;
    const double scale = -kappa / std::pow(h, gamma);
    for (double& x : w) x *= scale;
    p->colx = w;
    p->sigma = tau_spectrum(p->colx);
    const size_t L = next_pow2(2 * size_t(n_space));
    p->log_m = ilog2_exact(L / 2);
    std::vector<double> e = circulant_eigs(p->colx);
    for (double& x : e) x *= -dt / (2.0 * double(L));
    if (p->log_m == 13 || p->log_m == 14) {
      // the 2-CTA matvec's per-rank pair table (kernels_mv.cu): at double offset eigq_offset(M),
      // {eig[kap], eig[M - kap]} for task t of rank q, kap = q ? 2t + 1 : 2t + 2
      const size_t M = L / 2, H = M / 2;
      e.resize(fpc::eigq_offset(int(M)) + 4 * (H / 2), 0.0);
      double* eq = e.data() + fpc::eigq_offset(int(M));
      for (int q = 0; q < 2; ++q)
        for (size_t t = 0; t < H / 2; ++t) {
          const size_t kap = q ? 2 * t + 1 : 2 * t + 2;
          eq[2 * (q * (H / 2) + t)] = e[kap];
          eq[2 * (q * (H / 2) + t) + 1] = e[M - kap];
        }
    }
    p->d_eig = dalloc<double>(e.size());
    ck(cudaMemcpy(p->d_eig, e.data(), e.size() * sizeof(double), cudaMemcpyHostToDevice), "eig");
    *out = p;
  });
}

int fpc_problem_create_2d(fpc_context_t c, double gx, double gy, double kx, double ky, double h,
                          int n, int n_time, double dt, fpc_problem_t* out) {
  if (!c || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // RieszJacobian2D ctor (jacobian.hpp:58-69)
    if (!(kx > 0.0) || !(ky > 0.0))
      throw InvalidArg{"RieszJacobian2D: diffusion coefficients must be positive"};
    if (!(h > 0.0)) throw InvalidArg{"RieszJacobian2D: h must be positive"};
    if (n < 1) throw InvalidArg{"RieszJacobian2D: n_per_dim must be at least 1"};
    std::vector<double> wx = centred_weights(gx, n), wy = centred_weights(gy, n);
    if (n_time < 3) throw InvalidArg{"TimeStencil: need at least 3 time levels"};
    if (!(dt > 0.0)) throw InvalidArg{"AllAtOnceOperator: dt must be positive"};
    const bool pow2 = ilog2_exact(size_t(n_time)) >= 0 && n_time >= 4 && n_time <= 16384 &&
                      ilog2_exact(size_t(n) + 1) >= 0 && n >= 3 && n + 1 <= 4096;
    if (!pow2 && !(generic_sizes(n, n_time) && n >= 2))
      throw Unsupported{"B200 2D path: n_time a power of two in [4, 16384] and n_per_dim + 1 a power of two "
                        "in [4, 4096], or (any size) n_time <= 4096 and 2 <= n_per_dim <= 2047"};
    DeviceGuard g(c->device);
    fpc_problem_s* p = new_problem(c, n_time, dt);
    p->generic = pow2 ? 0 : 1;
    p->two_dim = 1;
    p->n = n;
    p->ns = n * n;
    p->colx = wx;
    p->coly = wy;
    p->sx = kx / std::pow(h, gx);  // jacobian.hpp:67-68
    p->sy = ky / std::pow(h, gy);
    // tau_spectrum_2d(tau(Tx), tau(Ty), -sx, -sy) (jacobian.hpp:96-98, tau.hpp:59-73)
    const std::vector<double> sgx = tau_spectrum(wx), sgy = tau_spectrum(wy);
    p->sigma.resize(size_t(n) * n);
    for (int ix = 0; ix < n; ++ix)
      for (int iy = 0; iy < n; ++iy)
        p->sigma[size_t(ix) * n + iy] = (-p->sx) * sgx[size_t(ix)] + (-p->sy) * sgy[size_t(iy)];
    const size_t L = next_pow2(2 * size_t(n));
    p->log_m = ilog2_exact(L / 2);
    // y = c - dt*A v with A = -sx Tx(x)I - sy I(x)Ty: the device factors are +dt*s*eig/(2L)
    std::vector<double> ey = circulant_eigs(wy), ex = circulant_eigs(wx);
    for (double& x : ey) x *= dt * p->sy / (2.0 * double(L));
    for (double& x : ex) x *= dt * p->sx / (2.0 * double(L));
    p->d_eig = dalloc<double>(ey.size());
    p->d_eig_x = dalloc<double>(ex.size());
    ck(cudaMemcpy(p->d_eig, ey.data(), ey.size() * sizeof(double), cudaMemcpyHostToDevice), "eig_y");
    ck(cudaMemcpy(p->d_eig_x, ex.data(), ex.size() * sizeof(double), cudaMemcpyHostToDevice), "eig_x");
    *out = p;
  });
}

static void release_problem(fpc_problem_s* p) {
  if (--p->refs > 0) return;
  fpc_context_s* c = p->ctx;
  {
    DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    cudaFree(p->d_eig);
    cudaFree(p->d_eig_x);
    cudaFree(p->d_in);
    cudaFree(p->d_out);
  }
  delete p;
  release_ctx(c);
}

int fpc_problem_destroy(fpc_problem_t p) {
  if (!p) return FPC_OK;
  release_problem(p);
  return FPC_OK;
}

int fpc_problem_dims(fpc_problem_t p, int* nt, int* ns, int* two_dim) {
  if (!p) return set_err(FPC_INVALID_ARGUMENT, "null problem");
  if (nt) *nt = p->nt;
  if (ns) *ns = p->ns;
  if (two_dim) *two_dim = p->two_dim;
  return FPC_OK;
}

int fpc_problem_first_column(fpc_problem_t p, int axis, double* out) {
  if (!p || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  const std::vector<double>& c = (axis == 1 && p->two_dim) ? p->coly : p->colx;
  std::memcpy(out, c.data(), c.size() * sizeof(double));
  return FPC_OK;
}

int fpc_problem_tau_sigma(fpc_problem_t p, double* out) {
  if (!p || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  std::memcpy(out, p->sigma.data(), p->sigma.size() * sizeof(double));
  return FPC_OK;
}

static void matvec_dev(fpc_problem_s* p, const double* v, double* y) {
  cudaStream_t st = p->ctx->stream;
  if (!p->two_dim) {
    LAUNCH("matvec_1d", st, fpc::launch_matvec_1d(v, y, p->ns, p->nt, p->log_m, p->d_eig, p->ctx->tw, st));
  } else {
    LAUNCH("matvec_2d", st, fpc::launch_matvec_2d(v, y, p->n, p->nt, p->log_m, p->d_eig, p->d_eig_x, p->ctx->tw, st));
  }
}

static void ensure_staging(fpc_problem_s* p) {
  if (!p->d_in) p->d_in = dalloc<double>(p->dim());
  if (!p->d_out) p->d_out = dalloc<double>(p->dim());
}

static void check_ptr(const void* ptr, const char* what) {
  if (!ptr) throw InvalidArg{std::string(what) + ": null pointer"};
}

static void check_dev_aligned(const void* ptr, const char* what) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
    throw InvalidArg{std::string(what) + ": device pointers must be 16-byte aligned"};
}

int fpc_matvec(fpc_problem_t p, const double* v, double* out, int where) {
  if (!p) return set_err(FPC_INVALID_ARGUMENT, "null problem");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_prob(p->mu);
    check_ptr(v, "fpc_matvec");
    check_ptr(out, "fpc_matvec");
    DeviceGuard g(p->ctx->device);
    const size_t n = p->dim();
    cudaStream_t st = p->ctx->stream;
    if (where == FPC_DEVICE) {
      check_dev_aligned(v, "fpc_matvec");
      check_dev_aligned(out, "fpc_matvec");
      if (v == out) throw InvalidArg{"fpc_matvec: input and output must be disjoint"};
      matvec_dev(p, v, out);
      return;
    }
    ensure_staging(p);
    upload(p->d_in, v, n * sizeof(double), st);
    matvec_dev(p, p->d_in, p->d_out);
    ck(cudaMemcpyAsync(out, p->d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

// all_at_once.hpp:66-80 (host; setup, not on the solve path)
int fpc_assemble_rhs(int nt, int ns, double dt, const double* f, const double* u0, double* b) {
  if (!f || !u0 || !b) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  if (nt < 2 || ns < 1) return set_err(FPC_INVALID_ARGUMENT, "assemble_rhs: size mismatch");
  const size_t NS = size_t(ns), NT = size_t(nt);
  for (size_t k = 0; k < NT; ++k)
    for (size_t i = 0; i < NS; ++i) b[k * NS + i] = dt * f[k * NS + i];
  for (size_t i = 0; i < NS; ++i) {
    b[i] += u0[i];
    b[NS + i] -= 0.5 * u0[i];
  }
  return FPC_OK;
}

// ---------------------------------------------------------------------------- plans
int fpc_plan_create(fpc_problem_t p, double alpha_in, fpc_plan_t* out) {
  if (!p || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    const int nt = p->nt;
    const double dt = p->dt;
    // PreconditionerKind::alpha_for (alpha_circulant.hpp:29-34)
    const double a = alpha_in <= 0.0 ? std::min(0.5, 0.5 * dt) : alpha_in;
    if (!(a > 0.0) || a > 1.0) throw InvalidArg{"PreconditionerKind: alpha must lie in (0, 1]"};
    auto* pl = new fpc_plan_s();
    pl->prob = p;
    pl->alpha = a;
    pl->n_warnings = a < 1e-8 ? 1 : 0;
    pl->lambda = alpha_lambda(a, nt);
    std::vector<double> sf(static_cast<size_t>(nt)), sb(static_cast<size_t>(nt));
    for (int k = 0; k < nt; ++k) {
      const double e = double(k) / double(nt);
      sf[size_t(k)] = std::pow(a, e);
      sb[size_t(k)] = std::pow(a, -e);
    }
    pl->solve_count = nt / 2 + 1;
    // singular-shift scan (alpha_circulant.hpp:110-123)
    double max_sigma = 0.0;
    for (double s : p->sigma) max_sigma = std::max(max_sigma, std::abs(s));
    double margin = std::numeric_limits<double>::infinity();
    for (int n = 0; n < pl->solve_count; ++n) {
      const cplx l = pl->lambda[size_t(n)];
      const double floor_ = 1e-14 * (std::abs(l) + dt * max_sigma);
      for (double s : p->sigma) {
        const double d = std::abs(l - dt * s);
        margin = std::min(margin, d);
        if (d <= floor_) {
          delete pl;
          throw RuntimeErr{"build_plan: an inner shifted system is numerically singular"};
        }
      }
    }
    pl->min_shift_margin = margin;
    DeviceGuard g(p->ctx->device);
    pl->d_sf = dalloc<double>(size_t(nt));
    pl->d_sb = dalloc<double>(size_t(nt));
    pl->d_lambda = dalloc<double2>(size_t(nt));  // all Nt: the full sweep solves every frequency
    // 2D: the transposed table sigma[iy][ix] follows the natural one (the column pass of the tau
    // solve reads sigma along ix for a fixed iy: contiguous in the transposed copy)
    pl->d_sigma = dalloc<double>(p->sigma.size() * (p->two_dim ? 2 : 1));
    pl->d_Z = dalloc<double2>(size_t(pl->solve_count) * size_t(p->ns));
    ck(cudaMemcpy(pl->d_sf, sf.data(), sf.size() * 8, cudaMemcpyHostToDevice), "sf");
    ck(cudaMemcpy(pl->d_sb, sb.data(), sb.size() * 8, cudaMemcpyHostToDevice), "sb");
    ck(cudaMemcpy(pl->d_lambda, pl->lambda.data(), size_t(nt) * 16, cudaMemcpyHostToDevice), "lambda");
    ck(cudaMemcpy(pl->d_sigma, p->sigma.data(), p->sigma.size() * 8, cudaMemcpyHostToDevice), "sigma");
    if (p->two_dim) {
      const size_t n = size_t(p->n);
      std::vector<double> st(p->sigma.size());
      for (size_t ix = 0; ix < n; ++ix)
        for (size_t iy = 0; iy < n; ++iy) st[iy * n + ix] = p->sigma[ix * n + iy];
      ck(cudaMemcpy(pl->d_sigma + p->sigma.size(), st.data(), st.size() * 8, cudaMemcpyHostToDevice), "sigmaT");
    }
    pl->scale_fwd = std::move(sf);
    pl->scale_bwd = std::move(sb);
    if (p->generic) {
      auto upload_c = [](const std::vector<cplx>& h) {
        double2* d = dalloc<double2>(h.size());
        ck(cudaMemcpy(d, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice), "chirp");
        return d;
      };
      const size_t nt_ = size_t(nt), P = 2 * (size_t(p->n) + 1);
      const auto ctf = bluestein_chirp(nt_, 1), cti = bluestein_chirp(nt_, -1), cds = bluestein_chirp(P, -1);
      pl->d_ctf = upload_c(ctf);
      pl->d_btf = upload_c(bluestein_filter(ctf, next_pow2(2 * nt_ - 1)));
      pl->d_cti = upload_c(cti);
      pl->d_bti = upload_c(bluestein_filter(cti, next_pow2(2 * nt_ - 1)));
      pl->d_cds = upload_c(cds);
      pl->d_bds = upload_c(bluestein_filter(cds, next_pow2(2 * P - 1)));
      pl->d_U = dalloc<double2>(nt_ * size_t(p->ns));
      const size_t seqs = p->two_dim ? nt_ * size_t(p->n) : nt_;  // full sweep: every frequency
      pl->d_D = dalloc<double2>(seqs * P);
    }
    ++p->refs;
    *out = pl;
  });
}

int fpc_plan_destroy(fpc_plan_t pl) {
  if (!pl) return FPC_OK;
  fpc_problem_s* p = pl->prob;
  {
    DeviceGuard g(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    for (double* b : pl->basis) cudaFree(b);
    for (double* b : pl->zbasis) cudaFree(b);
    for (void* q : {(void*)pl->d_sf, (void*)pl->d_sb, (void*)pl->d_lambda, (void*)pl->d_sigma,
                    (void*)pl->d_Z, (void*)pl->d_ZT, (void*)pl->d_z, (void*)pl->d_u, (void*)pl->d_r, (void*)pl->d_x,
                    (void*)pl->d_d, (void*)pl->d_b, (void*)pl->d_Zf, (void*)pl->d_ctf, (void*)pl->d_btf,
                    (void*)pl->d_cti, (void*)pl->d_bti, (void*)pl->d_cds, (void*)pl->d_bds, (void*)pl->d_U,
                    (void*)pl->d_D, (void*)pl->d_P})
      cudaFree(q);
  }
  delete pl;
  release_problem(p);
  return FPC_OK;
}

int fpc_plan_set_ordering(fpc_plan_t pl, int ordering) {
  if (!pl) return set_err(FPC_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    if (ordering != FPC_ORDER_REFERENCE && ordering != FPC_ORDER_COMMUTED)
      throw InvalidArg{"fpc_plan_set_ordering: bad ordering"};
    const fpc_problem_s* p = pl->prob;
    if (ordering == FPC_ORDER_COMMUTED && p->generic)
      throw Unsupported{"commuted ordering: power-of-two sizes only"};
    pl->ordering = ordering;
  });
}

int fpc_plan_info(fpc_plan_t pl, double* alpha, double* margin, int* solve_count, int* n_warn) {
  if (!pl) return set_err(FPC_INVALID_ARGUMENT, "null plan");
  if (alpha) *alpha = pl->alpha;
  if (margin) *margin = pl->min_shift_margin;
  if (solve_count) *solve_count = pl->solve_count;
  if (n_warn) *n_warn = pl->n_warnings;
  return FPC_OK;
}

int fpc_plan_scales(fpc_plan_t pl, double* scale_fwd, double* scale_bwd) {
  if (!pl || !scale_fwd || !scale_bwd) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  std::copy(pl->scale_fwd.begin(), pl->scale_fwd.end(), scale_fwd);
  std::copy(pl->scale_bwd.begin(), pl->scale_bwd.end(), scale_bwd);
  return FPC_OK;
}

int fpc_plan_lambda(fpc_plan_t pl, double* out) {
  if (!pl || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  std::memcpy(out, pl->lambda.data(), pl->lambda.size() * sizeof(cplx));
  return FPC_OK;
}

// z = P^{-1} (s_in * v)  (alpha_circulant.hpp:137-199, half sweep)
// forward = true: z = P (s_in v) from the same factors (apply_forward, alpha_circulant.hpp:212-215;
// the reference runs it as a full sweep, which for real v equals the Hermitian half sweep).
static void pc_apply_full_dev(fpc_plan_s* pl, const double* v, double* z, double s_in, bool forward);

// Generic sizes (kernels_generic.cu): the reference ordering on a full [Nt][Ns] complex spectrum
// with Bluestein transforms -- time FFT (fft_inplace(+1), alpha_circulant.hpp:146-152), the tau
// solves as dst_lattice / divide / dst_lattice (tau.hpp:79-119; 2D rows then columns), the
// conjugate mirror for the half sweep (167-175), inverse time FFT and real output (176-198),
// with the imaginary-residue guard for the full sweep.  apply_forward is the full sweep.
static void pc_apply_generic(fpc_plan_s* pl, const double* v, double* z, double s_in, bool forward) {
  fpc_problem_s* p = pl->prob;
  fpc_context_s* c = p->ctx;
  cudaStream_t st = c->stream;
  const int nt = p->nt, ns = p->ns, n = p->n, H = nt / 2 + 1;
  const bool full = forward || pl->sweep_mode == FPC_SWEEP_FULL;
  const long long act = full ? nt : H;
  const int mode = forward ? 2 : 1;
  LAUNCH("gen_time", st, fpc::launch_gen_time_in(v, pl->d_U, ns, nt, pl->d_sf, s_in, st));
  LAUNCH("gen_time", st, fpc::launch_bluestein(pl->d_U, nt, ns, ns, 0, 1, ns, pl->d_ctf, pl->d_btf, c->tw, st, 1));
  if (!p->two_dim) {
    LAUNCH("gen_tau", st, fpc::launch_gen_dst(pl->d_U, pl->d_D, n, act, 1, ns, 0, 1, pl->d_cds, pl->d_bds, c->tw, mode,
                                              1, ns, pl->d_lambda, pl->d_sigma, p->dt, st));
    LAUNCH("gen_tau", st, fpc::launch_gen_dst(pl->d_U, pl->d_D, n, act, 1, ns, 0, 1, pl->d_cds, pl->d_bds, c->tw, 0,
                                              1, ns, pl->d_lambda, pl->d_sigma, p->dt, st));
  } else {
    const long long nn = (long long)n * n, cnt = act * n;
    auto rows = [&](int md) {  // DST over iy of every (frequency, ix) row
      LAUNCH("gen_tau", st, fpc::launch_gen_dst(pl->d_U, pl->d_D, n, cnt, 1, n, 0, 1, pl->d_cds, pl->d_bds, c->tw, md,
                                                n, nn, pl->d_lambda, pl->d_sigma, p->dt, st));
    };
    auto cols = [&](int md) {  // DST over ix of every (frequency, iy) column
      LAUNCH("gen_tau", st, fpc::launch_gen_dst(pl->d_U, pl->d_D, n, cnt, n, nn, 1, n, pl->d_cds, pl->d_bds, c->tw, md,
                                                n, nn, pl->d_lambda, pl->d_sigma, p->dt, st));
    };
    rows(0);
    cols(mode);
    rows(0);
    cols(0);
  }
  if (!full) LAUNCH("gen_time", st, fpc::launch_gen_mirror(pl->d_U, nt, ns, H, st));
  LAUNCH("gen_time", st, fpc::launch_bluestein(pl->d_U, nt, ns, ns, 0, 1, ns, pl->d_cti, pl->d_bti, c->tw, st, -1));
  if (!full) {
    LAUNCH("gen_time", st, fpc::launch_gen_time_out(pl->d_U, z, ns, nt, pl->d_sb, st));
    return;
  }
  LAUNCH("gen_time", st, fpc::launch_gen_time_out_guard(pl->d_U, z, ns, nt, pl->d_sb, c->partial, st));
  LAUNCH("reduce", st, fpc::launch_reduce(c->partial, 2, 2, c->dscal + 960, false, st));
  ck(cudaMemcpyAsync(c->hpin + 960, c->dscal + 960, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  const double im2 = c->hpin[960], tot2 = c->hpin[961];
  if (tot2 > 0.0 && std::sqrt(im2) > 1e-10 * std::sqrt(tot2))
    throw RuntimeErr{"alpha-circulant action: imaginary residue exceeds 1e-10 of the output norm"};
}

// out = S (s_in v) for nlev (even) time levels: the spatial DST-I of every level (commuted ordering,
// SURVEY §8(f)1; dst.hpp:21-43 per level, tau.hpp:79-96 rows then columns in 2D).  1D with
// n_space + 1 <= 8192: the fused pair kernel; otherwise levels (2j, 2j+1) packed as one complex
// level, the complex row DSTs (1D: cluster kernels; 2D: rows then columns), unpacked.
static void dst_levels_dev(fpc_plan_s* pl, const double* v, double* out, int nlev, double s_in) {
  fpc_problem_s* p = pl->prob;
  cudaStream_t st = p->ctx->stream;
  if (!p->two_dim && p->ns + 1 <= 8192) {
    LAUNCH("dst_pairs", st, fpc::launch_dst_pairs(v, out, p->ns, nlev, s_in, p->ctx->tw, st));
    return;
  }
  if (!pl->d_P) pl->d_P = dalloc<double2>(size_t(p->nt / 2) * size_t(p->ns) + 1);
  LAUNCH("dst_pairs", st, fpc::launch_pack_pairs(v, pl->d_P, p->ns, nlev, s_in, st));
  if (!p->two_dim) {
    LAUNCH("dst_pairs", st, fpc::launch_dst_large(pl->d_P, p->ns, nlev / 2, p->ctx->tw, st));
  } else {
    LAUNCH("dst_pairs", st, fpc::launch_dst_rows(pl->d_P, p->n, (nlev / 2) * p->n, p->ctx->tw, st));
    LAUNCH("dst_pairs", st, fpc::launch_dst_cols_2d(pl->d_P, p->n, nlev / 2, p->ctx->tw, st));
  }
  LAUNCH("dst_pairs", st, fpc::launch_unpack_pairs(pl->d_P, out, p->ns, nlev, st));
}

static void pc_apply_dev(fpc_plan_s* pl, const double* v, double* z, double s_in,
                         bool forward = false) {
  if (pl->prob->generic) {
    pc_apply_generic(pl, v, z, s_in, forward);
    return;
  }
  if (pl->sweep_mode == FPC_SWEEP_FULL) {
    pc_apply_full_dev(pl, v, z, s_in, forward);
    return;
  }
  fpc_problem_s* p = pl->prob;
  cudaStream_t st = p->ctx->stream;
  if (pl->ordering == FPC_ORDER_COMMUTED) {
    // S per time level -> per-column time solve -> S per time level
    double* U = reinterpret_cast<double*>(pl->d_Z);
    dst_levels_dev(pl, v, U, p->nt, s_in);
    LAUNCH("time_solve", st,
           fpc::launch_time_solve(U, U, p->ns, p->nt, pl->d_sf, pl->d_sb, 1.0, pl->d_lambda, pl->d_sigma, p->dt,
                                  p->ctx->tw, st, forward));
    dst_levels_dev(pl, U, z, p->nt, 1.0);
    return;
  }
  LAUNCH("time_fwd", st, fpc::launch_time_fwd(v, pl->d_Z, p->ns, p->nt, pl->d_sf, s_in, p->ctx->tw, st));
  if (!p->two_dim)
    LAUNCH("tau_solve_1d", st,
           fpc::launch_tau_solve_1d(pl->d_Z, p->ns, pl->solve_count, pl->d_lambda, pl->d_sigma, p->dt,
                                    p->ctx->tw, st, forward));
  else {
    if (p->n == 255 && !pl->d_ZT) pl->d_ZT = dalloc<double2>(size_t(pl->solve_count) * size_t(p->ns));
    LAUNCH("tau_solve_2d", st,
           fpc::launch_tau_solve_2d(pl->d_Z, p->n, pl->solve_count, pl->d_lambda, pl->d_sigma, p->dt,
                                    p->ctx->tw, st, forward, pl->d_ZT));
  }
  LAUNCH("time_inv", st, fpc::launch_time_inv(pl->d_Z, z, p->ns, p->nt, pl->d_sb, p->ctx->tw, st));
}

// InnerSweep::full (alpha_circulant.hpp:158-159): all Nt frequency rows solved, complex inverse
// time FFT, and the imaginary-residue guard of alpha_circulant.hpp:196-198 (synchronous).
static void pc_apply_full_dev(fpc_plan_s* pl, const double* v, double* z, double s_in, bool forward) {
  fpc_problem_s* p = pl->prob;
  fpc_context_s* c = p->ctx;
  cudaStream_t st = c->stream;
  if (p->nt > 8192) throw Unsupported{"InnerSweep::full supports n_time <= 8192"};
  if (!pl->d_Zf) pl->d_Zf = dalloc<double2>(size_t(p->nt) * size_t(p->ns));
  LAUNCH("time_fwd", st, fpc::launch_time_fwd(v, pl->d_Zf, p->ns, p->nt, pl->d_sf, s_in, c->tw, st));
  LAUNCH("mirror_fill", st, fpc::launch_mirror_fill(pl->d_Zf, p->ns, p->nt, st));
  if (!p->two_dim)
    LAUNCH("tau_solve_1d", st,
           fpc::launch_tau_solve_1d(pl->d_Zf, p->ns, p->nt, pl->d_lambda, pl->d_sigma, p->dt, c->tw, st, forward));
  else
    LAUNCH("tau_solve_2d", st,
           fpc::launch_tau_solve_2d(pl->d_Zf, p->n, p->nt, pl->d_lambda, pl->d_sigma, p->dt, c->tw, st, forward));
  LAUNCH("time_inv_full", st, fpc::launch_time_inv_full(pl->d_Zf, z, p->ns, p->nt, pl->d_sb, c->tw, c->partial, st));
  LAUNCH("reduce", st, fpc::launch_reduce(c->partial, 2, 2, c->dscal + 960, false, st));
  ck(cudaMemcpyAsync(c->hpin + 960, c->dscal + 960, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  const double im2 = c->hpin[960], tot2 = c->hpin[961];
  if (tot2 > 0.0 && std::sqrt(im2) > 1e-10 * std::sqrt(tot2))
    throw RuntimeErr{"alpha-circulant action: imaginary residue exceeds 1e-10 of the output norm"};
}

int fpc_pc_apply(fpc_plan_t pl, const double* v, double* out, int sweep, int where) {
  if (!pl) return set_err(FPC_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    check_ptr(v, "fpc_pc_apply");
    check_ptr(out, "fpc_pc_apply");
    if (sweep != FPC_SWEEP_HALF && sweep != FPC_SWEEP_FULL) throw InvalidArg{"fpc_pc_apply: bad sweep"};
    pl->sweep_mode = sweep;
    fpc_problem_s* p = pl->prob;
    DeviceGuard g(p->ctx->device);
    const size_t n = p->dim();
    cudaStream_t st = p->ctx->stream;
    if (where == FPC_DEVICE) {
      check_dev_aligned(v, "fpc_pc_apply");
      check_dev_aligned(out, "fpc_pc_apply");
      pc_apply_dev(pl, v, out, 1.0);
      return;
    }
    ensure_staging(p);
    upload(p->d_in, v, n * sizeof(double), st);
    pc_apply_dev(pl, p->d_in, p->d_out, 1.0);
    ck(cudaMemcpyAsync(out, p->d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

int fpc_pc_forward(fpc_plan_t pl, const double* v, double* out, int where) {
  if (!pl) return set_err(FPC_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    check_ptr(v, "fpc_pc_forward");
    check_ptr(out, "fpc_pc_forward");
    // apply_forward is the full sweep in the reference (alpha_circulant.hpp:212-215)
    pl->sweep_mode = pl->prob->nt <= 8192 ? FPC_SWEEP_FULL : FPC_SWEEP_HALF;
    fpc_problem_s* p = pl->prob;
    DeviceGuard g(p->ctx->device);
    const size_t n = p->dim();
    cudaStream_t st = p->ctx->stream;
    if (where == FPC_DEVICE) {
      check_dev_aligned(v, "fpc_pc_forward");
      check_dev_aligned(out, "fpc_pc_forward");
      pc_apply_dev(pl, v, out, 1.0, true);
      return;
    }
    ensure_staging(p);
    upload(p->d_in, v, n * sizeof(double), st);
    pc_apply_dev(pl, p->d_in, p->d_out, 1.0, true);
    ck(cudaMemcpyAsync(out, p->d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

// ---------------------------------------------------------------------------- GMRES
namespace {

struct GmresState {
  fpc_plan_s* pl;
  fpc_context_s* ctx;
  size_t n;
  cudaStream_t st;
  std::vector<double> scales;  // basis[i] holds V_i / scales[i]... V_i = scales[i] * basis[i]
  int reorth = 0;
};

double* basis_buf(fpc_plan_s* pl, size_t i, size_t n) {
  while (pl->basis.size() <= i) pl->basis.push_back(dalloc<double>(n + 2));
  return pl->basis[i];
}

// Slot i of the preconditioned basis Z (z_i = P^{-1} V_i), or nullptr when keeping it would
// crowd out the Krylov basis: the basis slots the solve may still need (up to `basis_need`) plus
// 1 GiB of headroom must stay free.  Config 3 (8.6 GB vectors, GMRES(10)) does not keep Z.
double* zbasis_buf(fpc_plan_s* pl, size_t i, size_t n, size_t basis_need) {
  if (pl->zbasis.size() > i) return pl->zbasis[i];
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return nullptr;
  const size_t vec = (n + 2) * sizeof(double);
  const size_t more_basis = basis_need > pl->basis.size() ? basis_need - pl->basis.size() : 0;
  while (pl->zbasis.size() <= i) {
    if (free_b < vec * (more_basis + 1) + (size_t(1) << 30)) return nullptr;
    void* q = nullptr;
    if (cudaMalloc(&q, vec) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    pl->zbasis.push_back(static_cast<double*>(q));
    free_b -= vec;
  }
  return pl->zbasis[i];
}

// h[col0..col0+nv) (+ norm) into ctx->dscal[out_off...] via dots + deterministic reduce
void dots_into(GmresState& S, const std::vector<const double*>& V, int nv, const double* w,
               bool with_norm, int out_off) {
  fpc_context_s* c = S.ctx;
  const int stride = fpc_context_s::kPartialStride;
  if (nv == 0) {
    fpc::VecSet vs{};
    LAUNCH("dots", S.st, fpc::launch_dots(vs, 0, w, S.n, c->partial, stride, 0, true, S.st));
  }
  for (int g0 = 0; g0 < nv; g0 += 8) {
    const int cnt = std::min(8, nv - g0);
    fpc::VecSet vs{};
    for (int i = 0; i < cnt; ++i) {
      vs.v[i] = V[size_t(g0 + i)];
      vs.s[i] = S.scales[size_t(g0 + i)];
    }
    const bool last = g0 + cnt == nv;
    // the norm accumulator goes right after the last group's columns
    LAUNCH("dots", S.st, fpc::launch_dots(vs, cnt, w, S.n, c->partial, stride, g0, with_norm && last, S.st));
  }
  const int count = nv + (with_norm ? 1 : 0);
  LAUNCH("reduce", S.st, fpc::launch_reduce(c->partial, stride, count, c->dscal + out_off, false, S.st));
}

}  // namespace

static void gmres_inner(fpc_plan_s* pl, const double* b, double* x, double tol, int max_iter,
                        int* conv, int* steps_out, std::vector<double>& hist, double* last_rel,
                        int* reorth_count) {
  fpc_problem_s* p = pl->prob;
  fpc_context_s* c = p->ctx;
  GmresState S{pl, c, p->dim(), c->stream, {}, 0};
  const size_t n = S.n;
  *conv = 0;
  *steps_out = 0;
  // ||b||
  dots_into(S, {}, 0, b, true, 0);
  ck(cudaMemcpyAsync(c->hpin, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, S.st), "D2H");
  ck(cudaStreamSynchronize(S.st), "sync");
  const double norm_b = std::sqrt(c->hpin[0]);
  if (norm_b == 0.0) {
    ck(cudaMemsetAsync(x, 0, n * sizeof(double), S.st), "memset");
    *conv = 1;
    return;
  }
  std::vector<const double*> V;
  V.push_back(b);
  S.scales.push_back(1.0 / norm_b);
  std::vector<std::vector<double>> hcols;
  std::vector<double> gc, gs, g;
  g.push_back(norm_b);
  if (!pl->d_z) pl->d_z = dalloc<double>(n + 2);
  const double reorth_threshold = 0.70710678118654752;
  int steps = 0;
  // z_j = P^{-1} V_j is kept (when memory allows) so that x = Z y needs no extra preconditioner
  // apply: the reference forms x = P^{-1}(V y) (krylov.hpp:180-183); by linearity both are the same
  // x up to rounding, and Z costs no extra traffic (z_j is written by the PC apply either way).
  bool keep_z = true;
  for (int j = 0; j < max_iter; ++j) {
    double* zj = keep_z ? zbasis_buf(pl, size_t(j), n, size_t(max_iter)) : nullptr;
    if (!zj) {
      keep_z = false;
      zj = pl->d_z;
    }
    pc_apply_dev(pl, V[size_t(j)], zj, S.scales[size_t(j)]);
    double* w = basis_buf(pl, size_t(j), n);  // basis slot j holds V_{j+1} (V_0 = b)
    matvec_dev(p, zj, w);
    const int nv = j + 1;
    // CGS pass: h_i = <V_i, w>, norm_before^2
    dots_into(S, V, nv, w, true, 0);
    // copy pointer + scale tables for the update kernel
    std::vector<const double*> vp(V.begin(), V.end());
    ck(cudaMemcpyAsync(c->dvptr, vp.data(), vp.size() * sizeof(double*), cudaMemcpyHostToDevice, S.st),
       "vptr");
    ck(cudaMemcpyAsync(c->dscales, S.scales.data(), S.scales.size() * sizeof(double),
                       cudaMemcpyHostToDevice, S.st),
       "scales");
    std::vector<double> h(size_t(j) + 2, 0.0);
    double norm_before = 0.0, norm_w = 0.0;
    const int stride = fpc_context_s::kPartialStride;
    if (nv <= fpc::kMaxFused) {
      // fused: w' = w - V h and, in the same pass, c = V^T w' and ||w'||^2
      fpc::VecSetN vs{};
      for (int i = 0; i < nv; ++i) {
        vs.v[i] = V[size_t(i)];
        vs.s[i] = S.scales[size_t(i)];
      }
      LAUNCH("update_dots", S.st, fpc::launch_update_dots(vs, nv, c->dscal, w, n, c->partial, stride, S.st));
      LAUNCH("reduce", S.st, fpc::launch_reduce(c->partial, stride, nv + 1, c->dscal + 256, false, S.st));
      ck(cudaMemcpyAsync(c->hpin, c->dscal, size_t(nv + 1) * sizeof(double), cudaMemcpyDeviceToHost, S.st),
         "D2H");
      ck(cudaMemcpyAsync(c->hpin + 256, c->dscal + 256, size_t(nv + 1) * sizeof(double),
                         cudaMemcpyDeviceToHost, S.st),
         "D2H");
      ck(cudaStreamSynchronize(S.st), "sync");
      for (int i = 0; i <= j; ++i) h[size_t(i)] = c->hpin[i];
      norm_before = std::sqrt(c->hpin[nv]);
      norm_w = std::sqrt(c->hpin[256 + nv]);
      if (norm_w < reorth_threshold * norm_before) {  // krylov.hpp:123-130 (dots already done)
        ++*reorth_count;
        LAUNCH("update", S.st, fpc::launch_update(c->dvptr, c->dscales, c->dscal + 256, nv, w, n, c->partial, S.st));
        LAUNCH("reduce", S.st, fpc::launch_reduce(c->partial, 1, 1, c->dscal + 512, false, S.st));
        ck(cudaMemcpyAsync(c->hpin + 512, c->dscal + 512, sizeof(double), cudaMemcpyDeviceToHost, S.st), "D2H");
        ck(cudaStreamSynchronize(S.st), "sync");
        for (int i = 0; i <= j; ++i) h[size_t(i)] += c->hpin[256 + i];
        norm_w = std::sqrt(c->hpin[512]);
      }
    } else {
      LAUNCH("update", S.st, fpc::launch_update(c->dvptr, c->dscales, c->dscal, nv, w, n, c->partial, S.st));
      LAUNCH("reduce", S.st, fpc::launch_reduce(c->partial, 1, 1, c->dscal + 512, false, S.st));
      ck(cudaMemcpyAsync(c->hpin, c->dscal, size_t(nv + 1) * sizeof(double), cudaMemcpyDeviceToHost, S.st),
         "D2H");
      ck(cudaMemcpyAsync(c->hpin + 512, c->dscal + 512, sizeof(double), cudaMemcpyDeviceToHost, S.st), "D2H");
      ck(cudaStreamSynchronize(S.st), "sync");
      for (int i = 0; i <= j; ++i) h[size_t(i)] = c->hpin[i];
      norm_before = std::sqrt(c->hpin[nv]);
      norm_w = std::sqrt(c->hpin[512]);
      if (norm_w < reorth_threshold * norm_before) {  // krylov.hpp:123-130
        ++*reorth_count;
        dots_into(S, V, nv, w, false, 256);
        LAUNCH("update", S.st, fpc::launch_update(c->dvptr, c->dscales, c->dscal + 256, nv, w, n, c->partial, S.st));
        LAUNCH("reduce", S.st, fpc::launch_reduce(c->partial, 1, 1, c->dscal + 512, false, S.st));
        ck(cudaMemcpyAsync(c->hpin + 256, c->dscal + 256, size_t(nv) * sizeof(double),
                           cudaMemcpyDeviceToHost, S.st),
           "D2H");
        ck(cudaMemcpyAsync(c->hpin + 512, c->dscal + 512, sizeof(double), cudaMemcpyDeviceToHost, S.st), "D2H");
        ck(cudaStreamSynchronize(S.st), "sync");
        for (int i = 0; i <= j; ++i) h[size_t(i)] += c->hpin[256 + i];
        norm_w = std::sqrt(c->hpin[512]);
      }
    }
    h[size_t(j) + 1] = norm_w;
    // Givens (krylov.hpp:133-151)
    for (int i = 0; i < j; ++i) {
      const double hi = h[size_t(i)], hi1 = h[size_t(i) + 1];
      h[size_t(i)] = gc[size_t(i)] * hi + gs[size_t(i)] * hi1;
      h[size_t(i) + 1] = -gs[size_t(i)] * hi + gc[size_t(i)] * hi1;
    }
    const double hj = h[size_t(j)], hj1 = h[size_t(j) + 1];
    const double rad = std::hypot(hj, hj1);
    const double cs = rad > 0.0 ? hj / rad : 1.0;
    const double sn = rad > 0.0 ? hj1 / rad : 0.0;
    gc.push_back(cs);
    gs.push_back(sn);
    h[size_t(j)] = rad;
    h[size_t(j) + 1] = 0.0;
    g.push_back(-sn * g[size_t(j)]);
    g[size_t(j)] *= cs;
    hcols.push_back(h);
    steps = j + 1;
    const double rel = std::abs(g[size_t(j) + 1]) / norm_b;
    hist.push_back(rel);
    *last_rel = rel;
    if (rel <= tol) {
      *conv = 1;
      break;
    }
    if (norm_w <= 1e-14 * std::max(1.0, norm_before)) break;  // krylov.hpp:160-165
    V.push_back(w);
    S.scales.push_back(1.0 / norm_w);
  }
  // back substitution (krylov.hpp:171-179), u = V y, x = P^{-1} u
  std::vector<double> y(size_t(steps), 0.0);
  for (int i = steps - 1; i >= 0; --i) {
    double s = g[size_t(i)];
    for (int k = i + 1; k < steps; ++k) s -= hcols[size_t(k)][size_t(i)] * y[size_t(k)];
    y[size_t(i)] = s / hcols[size_t(i)][size_t(i)];
  }
  std::memcpy(c->hpin + 600, y.data(), y.size() * sizeof(double));
  ck(cudaMemcpyAsync(c->dscal + 600, c->hpin + 600, y.size() * sizeof(double), cudaMemcpyHostToDevice, S.st),
     "y");
  if (keep_z && steps > 0) {
    // x = Z y (z_i already carries the basis scale)
    std::vector<const double*> zp(pl->zbasis.begin(), pl->zbasis.begin() + steps);
    std::vector<double> ones(size_t(steps), 1.0);
    ck(cudaMemcpyAsync(c->dvptr, zp.data(), zp.size() * sizeof(double*), cudaMemcpyHostToDevice, S.st), "vptr");
    std::memcpy(c->hpin + 1024, ones.data(), ones.size() * sizeof(double));
    ck(cudaMemcpyAsync(c->dscales, c->hpin + 1024, size_t(steps) * sizeof(double), cudaMemcpyHostToDevice, S.st),
       "scales");
    LAUNCH("lincomb", S.st, fpc::launch_lincomb(c->dvptr, c->dscales, c->dscal + 600, steps, x, n, S.st));
  } else {
    // u = V y lives in the z buffer (z is dead after the loop): one 8N buffer less at config 3
    double* u = pl->d_z;
    std::vector<const double*> vp(V.begin(), V.begin() + steps);
    ck(cudaMemcpyAsync(c->dvptr, vp.data(), vp.size() * sizeof(double*), cudaMemcpyHostToDevice, S.st), "vptr");
    ck(cudaMemcpyAsync(c->dscales, S.scales.data(), size_t(steps) * sizeof(double), cudaMemcpyHostToDevice, S.st),
       "scales");
    LAUNCH("lincomb", S.st, fpc::launch_lincomb(c->dvptr, c->dscales, c->dscal + 600, steps, u, n, S.st));
    pc_apply_dev(pl, u, x, 1.0);
  }
  *steps_out = steps;
  ck(cudaStreamSynchronize(S.st), "sync");  // hpin reuse boundary
}

// GMRES with delayed re-orthogonalisation (classical Gram-Schmidt twice, the second pass lagged
// one step; the low-synchronisation DCGS2 of Bielich et al., in the Arnoldi form).  Same Krylov
// space and the same least-squares problem as the reference's gmres_right (krylov.hpp:83-192:
// Gram-Schmidt with re-orthogonalisation, which fires on every step of this preconditioned
// system); per step the basis is read twice instead of three times:
//   iteration j >= 1 has the once-orthogonalised candidate u~ (norm nu) of v_j in a buffer and
//   runs w = A P^{-1} (u~/nu), then
//   Q1  one pass: a = V^T u~, b = V^T w, <u~,w>, ||u~||^2, ||w||^2          (one sync)
//       host: v_j = (u~ - V a)/rho, rho^2 = ||u~||^2 - ||a||^2 finalises Hessenberg column j-1;
//       A P^{-1} v_j = (nu w - V_{0..j} H a)/rho by the Arnoldi relation, so the projections
//       e = V_{0..j}^T A P^{-1} v_j follow from a, b and H without touching the vectors;
//   Q2  one pass: u~ <- rho v_j, w <- A P^{-1} v_j - V_{0..j} e (the next candidate), ||w||^2.
// The step's convergence test uses the candidate's norm for H_{j+1,j}; the next Q1 replaces it by
// the re-orthogonalised value and redoes that Givens rotation (a 1e-13-relative change here).
// With Z kept, z~_j = P^{-1}(u~_j/nu_j) and x = Z~ (T y), T upper triangular from the same a's.
static void gmres_inner_lagged(fpc_plan_s* pl, const double* b, double* x, double tol, int max_iter,
                               int* conv, int* steps_out, std::vector<double>& hist, double* last_rel,
                               int* reorth_count) {
  fpc_problem_s* p = pl->prob;
  fpc_context_s* c = p->ctx;
  GmresState S{pl, c, p->dim(), c->stream, {}, 0};
  const size_t n = S.n;
  cudaStream_t st = S.st;
  const int stride = fpc_context_s::kPartialStride;
  *conv = 0;
  *steps_out = 0;
  dots_into(S, {}, 0, b, true, 0);
  ck(cudaMemcpyAsync(c->hpin, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  const double norm_b = std::sqrt(c->hpin[0]);
  if (norm_b == 0.0) {
    ck(cudaMemsetAsync(x, 0, n * sizeof(double), st), "memset");
    *conv = 1;
    return;
  }
  if (!pl->d_z) pl->d_z = dalloc<double>(n + 2);
  // V[i]: buffer of basis vector i (V[0] = b, read only); v_i = sc[i] * V[i] once final
  std::vector<double*> V{const_cast<double*>(b)};
  std::vector<double> sc{1.0 / norm_b};
  // Implicit re-orthogonalisation (default): the stored vectors V[k] are never rewritten; the
  // orthonormal basis is v_k = sum_{i<=k} Sc[k][i] V[i], with the lagged second Gram-Schmidt pass
  // of vector k entering Sc[k] instead of a U <- U - V a sweep (same vectors, two basis passes less
  // per step: no read and no write of U in Q2).  Dots against the stored vectors are mapped to the
  // orthonormal basis by Sc^T, update coefficients back by Sc.  FPC_GS_IMPLICIT=0: rewrite U.
  static const bool implicit = [] {
    const char* e = std::getenv("FPC_GS_IMPLICIT");
    return !(e && e[0] == '0');
  }();
  std::vector<std::vector<double>> Sc{{1.0 / norm_b}};
  std::vector<std::vector<double>> R;   // raw Hessenberg columns (final, except the newest)
  std::vector<std::vector<double>> T;   // T[j][i]: Z_j = sum_i T[j][i] z~_i
  std::vector<double> gc, gs, g{norm_b}, g_pre, nb_before;
  bool keep_z = true;
  std::vector<double*> zt;
  auto rotate_column = [&](int j, std::vector<double> h) {
    // apply the final rotations 0..j-1 to raw column j, then form rotation j; g[j], g[j+1] from g_pre[j]
    for (int i = 0; i < j; ++i) {
      const double hi = h[size_t(i)], hi1 = h[size_t(i) + 1];
      h[size_t(i)] = gc[size_t(i)] * hi + gs[size_t(i)] * hi1;
      h[size_t(i) + 1] = -gs[size_t(i)] * hi + gc[size_t(i)] * hi1;
    }
    const double hj = h[size_t(j)], hj1 = h[size_t(j) + 1];
    const double rad = std::hypot(hj, hj1);
    const double cs = rad > 0.0 ? hj / rad : 1.0;
    const double sn = rad > 0.0 ? hj1 / rad : 0.0;
    if (gc.size() <= size_t(j)) {
      gc.push_back(cs);
      gs.push_back(sn);
      g_pre.push_back(g[size_t(j)]);
      g.push_back(0.0);
    } else {
      gc[size_t(j)] = cs;
      gs[size_t(j)] = sn;
    }
    g[size_t(j) + 1] = -sn * g_pre[size_t(j)];
    g[size_t(j)] = cs * g_pre[size_t(j)];
    h[size_t(j)] = rad;
    h[size_t(j) + 1] = 0.0;
    return h;
  };
  std::vector<std::vector<double>> Hr;  // rotated columns (for the back substitution)
  int steps = 0;
  double nu = 0.0;  // norm of the candidate in V[j]
  for (int j = 0; j < max_iter; ++j) {
    double* zj = keep_z ? zbasis_buf(pl, size_t(j), n, size_t(max_iter)) : nullptr;
    if (!zj) {
      keep_z = false;
      zj = pl->d_z;
    }
    zt.push_back(zj);
    double* W = basis_buf(pl, size_t(j), n);  // slot j holds basis vector j + 1
    pc_apply_dev(pl, V[size_t(j)], zj, j == 0 ? sc[0] : 1.0 / nu);
    matvec_dev(p, zj, W);
    std::vector<double> col(size_t(j) + 2, 0.0);
    double norm_before = 0.0, nu_next = 0.0;
    if (j == 0) {
      // first vector: plain pass h_0 = <v_0, w>, w -= h_0 v_0 (v_0 = b/||b|| is exact)
      S.scales.assign(1, sc[0]);
      dots_into(S, {b}, 1, W, true, 0);
      ck(cudaMemcpyAsync(c->dvptr, V.data(), sizeof(double*), cudaMemcpyHostToDevice, st), "vptr");
      ck(cudaMemcpyAsync(c->dscales, sc.data(), sizeof(double), cudaMemcpyHostToDevice, st), "scales");
      LAUNCH("update", st, fpc::launch_update(c->dvptr, c->dscales, c->dscal, 1, W, n, c->partial, st));
      LAUNCH("reduce", st, fpc::launch_reduce(c->partial, 1, 1, c->dscal + 512, false, st));
      ck(cudaMemcpyAsync(c->hpin, c->dscal, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaMemcpyAsync(c->hpin + 512, c->dscal + 512, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      col[0] = c->hpin[0];
      norm_before = std::sqrt(c->hpin[1]);
      nu_next = std::sqrt(c->hpin[512]);
      T.push_back({1.0});
    } else {
      // Q1: a = V^T u~, b = V^T w (+ <u~,w>, ||u~||^2, ||w||^2)
      double* U = V[size_t(j)];
      for (int g0 = 0; g0 < j; g0 += 16) {
        const int cnt = std::min(16, j - g0);
        fpc::VecSet16 vs{};
        for (int i = 0; i < cnt; ++i) {
          vs.v[i] = V[size_t(g0 + i)];
          vs.s[i] = implicit ? 1.0 : sc[size_t(g0 + i)];
        }
        LAUNCH("dots2", st, fpc::launch_dots2(vs, cnt, U, W, n, c->partial, stride, g0, g0 == 0, st));
      }
      LAUNCH("reduce", st, fpc::launch_reduce_dots2(c->partial, stride, j, c->dscal, st));
      ck(cudaMemcpyAsync(c->hpin, c->dscal, (fpc::kDots2X + 3) * sizeof(double), cudaMemcpyDeviceToHost, st),
         "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      std::vector<double> a(static_cast<size_t>(j)), bb(static_cast<size_t>(j));
      double aa = 0.0, ab = 0.0;
      for (int i = 0; i < j; ++i) {
        if (implicit) {  // <v_i, .> = sum_l Sc[i][l] <V[l], .>
          double sa = 0.0, sb = 0.0;
          for (int l = 0; l <= i; ++l) {
            sa += Sc[size_t(i)][size_t(l)] * c->hpin[l];
            sb += Sc[size_t(i)][size_t(l)] * c->hpin[fpc::kDots2B + l];
          }
          a[size_t(i)] = sa;
          bb[size_t(i)] = sb;
        } else {
          a[size_t(i)] = c->hpin[i];
          bb[size_t(i)] = c->hpin[fpc::kDots2B + i];
        }
        aa += a[size_t(i)] * a[size_t(i)];
        ab += a[size_t(i)] * bb[size_t(i)];
      }
      const double beta = c->hpin[fpc::kDots2X], uu = c->hpin[fpc::kDots2X + 1], ww = c->hpin[fpc::kDots2X + 2];
      const double rho = std::sqrt(std::max(uu - aa, 0.0));
      ++*reorth_count;
      // finalise column j-1 with the re-orthogonalised v_j and redo its rotation
      std::vector<double>& rc = R[size_t(j) - 1];
      for (int i = 0; i < j; ++i) rc[size_t(i)] += a[size_t(i)];
      rc[size_t(j)] = rho;
      Hr[size_t(j) - 1] = rotate_column(j - 1, rc);
      const double rel_c = std::abs(g[size_t(j)]) / norm_b;
      hist.back() = rel_c;
      *last_rel = rel_c;
      if (rel_c <= tol) {  // converged at step j after all (the estimate was just above tol)
        *conv = 1;
        break;
      }
      if (rho <= 1e-14 * std::max(1.0, nb_before[size_t(j) - 1])) break;  // krylov.hpp:160-165
      sc.push_back(1.0 / rho);
      if (implicit) {  // v_j = (V[j] - sum_l a_l v_l)/rho
        std::vector<double> sj(size_t(j) + 1, 0.0);
        for (int l = 0; l < j; ++l)
          for (int i = 0; i <= l; ++i) sj[size_t(i)] -= a[size_t(l)] * Sc[size_t(l)][size_t(i)] / rho;
        sj[size_t(j)] = 1.0 / rho;
        Sc.push_back(sj);
      }
      // T column j: Z_j = (nu z~_j - sum_l a_l Z_l)/rho
      std::vector<double> tj(size_t(j) + 1, 0.0);
      tj[size_t(j)] = nu / rho;
      for (int l = 0; l < j; ++l)
        for (int i = 0; i <= l; ++i) tj[size_t(i)] -= a[size_t(l)] * T[size_t(l)][size_t(i)] / rho;
      T.push_back(tj);
      // gg = H_{0..j, 0..j-1} a (Arnoldi relation), e = V_{0..j}^T A P^{-1} v_j
      std::vector<double> gg(size_t(j) + 1, 0.0);
      for (int l = 0; l < j; ++l)
        for (int k = 0; k <= l + 1; ++k) gg[size_t(k)] += R[size_t(l)][size_t(k)] * a[size_t(l)];
      for (int k = 0; k < j; ++k) col[size_t(k)] = (nu * bb[size_t(k)] - gg[size_t(k)]) / rho;
      col[size_t(j)] = (nu * (beta - ab) / rho - gg[size_t(j)]) / rho;
      // Q2: U <- U - V a (= rho v_j);  W <- cw W + cu U + V cd (= the next candidate)
      const double t = gg[size_t(j)] / rho + col[size_t(j)];
      const double cw = nu / rho, cu = -t / rho;
      // coefficient of v_k in the W update; implicit: mapped onto the stored vectors, cds = Sc cdt
      std::vector<double> cdt(static_cast<size_t>(j)), cds(static_cast<size_t>(j), 0.0);
      for (int k = 0; k < j; ++k) cdt[size_t(k)] = -gg[size_t(k)] / rho - col[size_t(k)] + t * a[size_t(k)] / rho;
      if (implicit)
        for (int k = 0; k < j; ++k)
          for (int i = 0; i <= k; ++i) cds[size_t(i)] += Sc[size_t(k)][size_t(i)] * cdt[size_t(k)];
      for (int g0 = 0; g0 < j || g0 == 0; g0 += fpc::kMaxUpd2) {
        const int cnt = std::min(fpc::kMaxUpd2, j - g0);
        fpc::Update2Args ua{};
        ua.cw = cw;
        ua.cu = cu;
        for (int i = 0; i < cnt; ++i) {
          const int k = g0 + i;
          ua.v[i] = V[size_t(k)];
          ua.ca[i] = implicit ? 0.0 : a[size_t(k)] * sc[size_t(k)];
          ua.cd[i] = implicit ? cds[size_t(k)] : cdt[size_t(k)] * sc[size_t(k)];
        }
        const bool last = g0 + cnt >= j;
        LAUNCH("update2", st, fpc::launch_update2(ua, cnt, g0 == 0, last, U, W, n, c->partial, st, implicit));
        if (last) break;
      }
      LAUNCH("reduce", st, fpc::launch_reduce(c->partial, 1, 1, c->dscal + 512, false, st));
      ck(cudaMemcpyAsync(c->hpin + 512, c->dscal + 512, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      nu_next = std::sqrt(c->hpin[512]);
      double e2 = 0.0;
      for (int k = 0; k <= j; ++k) e2 += col[size_t(k)] * col[size_t(k)];
      norm_before = std::sqrt(e2 + nu_next * nu_next);  // ||A P^{-1} v_j||
      (void)ww;
    }
    col[size_t(j) + 1] = nu_next;  // estimate until the next Q1 re-orthogonalises
    R.push_back(col);
    nb_before.push_back(norm_before);
    Hr.push_back(rotate_column(j, col));
    steps = j + 1;
    const double rel = std::abs(g[size_t(j) + 1]) / norm_b;
    hist.push_back(rel);
    *last_rel = rel;
    if (rel <= tol) {
      *conv = 1;
      break;
    }
    if (nu_next <= 1e-14 * std::max(1.0, norm_before)) break;
    V.push_back(W);
    nu = nu_next;
  }
  // back substitution (krylov.hpp:171-179) on the rotated columns
  std::vector<double> y(size_t(steps), 0.0);
  for (int i = steps - 1; i >= 0; --i) {
    double sacc = g[size_t(i)];
    for (int k = i + 1; k < steps; ++k) sacc -= Hr[size_t(k)][size_t(i)] * y[size_t(k)];
    y[size_t(i)] = sacc / Hr[size_t(i)][size_t(i)];
  }
  std::vector<double> coef(size_t(steps), 0.0), scales(size_t(steps), 1.0);
  std::vector<const double*> ptr(static_cast<size_t>(steps));
  if (keep_z) {
    // x = Z y = Z~ (T y)
    for (int jj = 0; jj < steps; ++jj)
      for (int i = 0; i <= jj; ++i) coef[size_t(i)] += T[size_t(jj)][size_t(i)] * y[size_t(jj)];
    for (int i = 0; i < steps; ++i) ptr[size_t(i)] = zt[size_t(i)];
  } else {
    for (int i = 0; i < steps; ++i) {
      coef[size_t(i)] = y[size_t(i)];
      scales[size_t(i)] = sc[size_t(i)];
      ptr[size_t(i)] = V[size_t(i)];
    }
    if (implicit) {  // V y = V~ (Sc y)
      std::fill(coef.begin(), coef.end(), 0.0);
      std::fill(scales.begin(), scales.end(), 1.0);
      for (int k = 0; k < steps; ++k)
        for (int i = 0; i <= k; ++i) coef[size_t(i)] += Sc[size_t(k)][size_t(i)] * y[size_t(k)];
    }
  }
  ck(cudaMemcpyAsync(c->dvptr, ptr.data(), ptr.size() * sizeof(double*), cudaMemcpyHostToDevice, st), "vptr");
  std::memcpy(c->hpin + 1024, scales.data(), scales.size() * sizeof(double));
  ck(cudaMemcpyAsync(c->dscales, c->hpin + 1024, scales.size() * sizeof(double), cudaMemcpyHostToDevice, st),
     "scales");
  std::memcpy(c->hpin + 600, coef.data(), coef.size() * sizeof(double));
  ck(cudaMemcpyAsync(c->dscal + 600, c->hpin + 600, coef.size() * sizeof(double), cudaMemcpyHostToDevice, st),
     "coef");
  if (keep_z) {
    LAUNCH("lincomb", st, fpc::launch_lincomb(c->dvptr, c->dscales, c->dscal + 600, steps, x, n, st));
  } else {
    double* u = pl->d_z;
    LAUNCH("lincomb", st, fpc::launch_lincomb(c->dvptr, c->dscales, c->dscal + 600, steps, u, n, st));
    pc_apply_dev(pl, u, x, 1.0);
  }
  *steps_out = steps;
  ck(cudaStreamSynchronize(st), "sync");
}

// GS scheme: FPC_GS=cgs2 selects the reference-shaped CGS + conditional re-orthogonalisation loop
static bool use_lagged_gs(int max_iter) {
  static const int mode = [] {
    const char* e = std::getenv("FPC_GS");
    return (e && std::string(e) == "cgs2") ? 0 : 1;
  }();
  return mode == 1 && max_iter <= 120;
}

static double resid_norm_dev(fpc_plan_s* pl, const double* b, const double* x) {
  fpc_problem_s* p = pl->prob;
  fpc_context_s* c = p->ctx;
  const size_t n = p->dim();
  if (!pl->d_z) pl->d_z = dalloc<double>(n + 2);
  double* r = pl->d_z;  // scratch; z is not live here
  matvec_dev(p, x, r);
  LAUNCH("resid", c->stream, fpc::launch_resid_norm(b, r, n, c->partial, c->stream));
  LAUNCH("reduce", c->stream, fpc::launch_reduce(c->partial, 1, 1, c->dscal + 900, false, c->stream));
  ck(cudaMemcpyAsync(c->hpin + 900, c->dscal + 900, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  return std::sqrt(c->hpin[900]);
}

// Host-path result copy: x (final once the Krylov loop ends) goes to the caller's buffer on a side
// stream while the main stream runs the true-residual check (krylov.hpp:188, a matvec and a norm,
// which only read x).  The caller synchronises the side stream before returning.
static void copy_out_async(fpc_context_s* c, double* host_x, const double* x, size_t n) {
  if (!c->aux) {
    ck(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&c->aux_ev, cudaEventDisableTiming), "cudaEventCreate");
  }
  ck(cudaEventRecord(c->aux_ev, c->stream), "event");
  ck(cudaStreamWaitEvent(c->aux, c->aux_ev, 0), "wait");
  ck(cudaMemcpyAsync(host_x, x, n * sizeof(double), cudaMemcpyDeviceToHost, c->aux), "D2H");
}

static void gmres_dev(fpc_plan_s* pl, const double* b, double* x, const fpc_solver_config& cfg,
                      fpc_report* rep, std::vector<double>& hist, double* host_x = nullptr) {
  fpc_problem_s* p = pl->prob;
  fpc_context_s* c = p->ctx;
  const size_t n = p->dim();
  double last_rel = -1.0;
  int reorth = 0;
  if (cfg.restart <= 0 || cfg.restart >= cfg.max_iter) {
    int conv = 0, steps = 0;
    (use_lagged_gs(cfg.max_iter) ? gmres_inner_lagged : gmres_inner)(pl, b, x, cfg.tol, cfg.max_iter, &conv, &steps,
                                                                     hist, &last_rel, &reorth);
    rep->converged = conv;
    rep->iterations = steps;
  } else {
    // GMRES(m): restart emulation of SURVEY §8(c) (same as oracle/fracpint_oracle.c orc_gmres)
    if (!pl->d_d) pl->d_d = dalloc<double>(n + 2);
    if (!pl->d_b) pl->d_b = dalloc<double>(n + 2);
    double* r = pl->d_b;  // current residual (rhs of the inner solve)
    ck(cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
    ck(cudaMemsetAsync(x, 0, n * sizeof(double), c->stream), "memset");
    // ||b||
    GmresState S{pl, c, n, c->stream, {}, 0};
    dots_into(S, {}, 0, b, true, 0);
    ck(cudaMemcpyAsync(c->hpin, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    const double norm_b = std::sqrt(c->hpin[0]);
    int budget = cfg.max_iter, total = 0, conv_all = 0;
    while (budget > 0) {
      dots_into(S, {}, 0, r, true, 0);
      ck(cudaMemcpyAsync(c->hpin, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
      ck(cudaStreamSynchronize(c->stream), "sync");
      const double norm_r = std::sqrt(c->hpin[0]);
      if (norm_r == 0.0) {
        conv_all = 1;
        break;
      }
      const int m = std::min(cfg.restart, budget);
      int conv = 0, steps = 0;
      const size_t h0 = hist.size();
      (use_lagged_gs(m) ? gmres_inner_lagged : gmres_inner)(pl, r, pl->d_d, cfg.tol * norm_b / norm_r, m, &conv, &steps,
                                                            hist, &last_rel, &reorth);
      for (size_t i = h0; i < hist.size(); ++i) hist[i] *= norm_r / norm_b;
      if (last_rel >= 0.0) last_rel *= norm_r / norm_b;
      LAUNCH("axpy", c->stream, fpc::launch_axpy(1.0, pl->d_d, x, n, c->stream));
      total += steps;
      budget -= steps;
      if (conv) {
        conv_all = 1;
        break;
      }
      if (steps == 0) break;
      ++rep->restarts;
      matvec_dev(p, x, r);
      LAUNCH("rsub", c->stream, fpc::launch_rsub(b, r, n, c->stream));
    }
    rep->converged = conv_all;
    rep->iterations = total;
  }
  rep->reorthogonalizations = reorth;
  rep->final_relative_residual = hist.empty() ? 1.0 : last_rel;
  if (host_x) copy_out_async(c, host_x, x, n);
  // fresh_relative_residual (krylov.hpp:64-75)
  GmresState S{pl, c, n, c->stream, {}, 0};
  dots_into(S, {}, 0, b, true, 0);
  ck(cudaMemcpyAsync(c->hpin, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  const double norm_b = std::sqrt(c->hpin[0]);
  if (norm_b == 0.0) {
    rep->final_relative_residual = 0.0;
    rep->true_relative_residual = 0.0;
    rep->converged = 1;
    return;
  }
  rep->true_relative_residual = resid_norm_dev(pl, b, x) / norm_b;
}

int fpc_gmres(fpc_plan_t pl, const double* b, double* x, const fpc_solver_config* cfg_in,
              fpc_report* rep, double* history, int history_cap, int where) {
  if (!pl || !rep) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    check_ptr(b, "fpc_gmres");
    check_ptr(x, "fpc_gmres");
    fpc_solver_config cfg{1e-9, 200, 0, FPC_SWEEP_HALF};
    if (cfg_in) cfg = *cfg_in;
    if (cfg.sweep != FPC_SWEEP_HALF && cfg.sweep != FPC_SWEEP_FULL) throw InvalidArg{"fpc_gmres: bad sweep"};
    pl->sweep_mode = cfg.sweep;
    if (cfg.max_iter < 0) throw InvalidArg{"gmres_right: max_iter must be non-negative"};
    // basis vectors live at once: one restart cycle (GMRES(m)), or the whole unrestarted solve
    const int basis_steps = (cfg.restart > 0 && cfg.restart < cfg.max_iter) ? cfg.restart : cfg.max_iter;
    if (basis_steps > 250) throw Unsupported{"B200 GMRES keeps at most 250 basis vectors per cycle"};
    fpc_problem_s* p = pl->prob;
    DeviceGuard g(p->ctx->device);
    const auto t0 = std::chrono::steady_clock::now();
    std::memset(rep, 0, sizeof *rep);
    std::vector<double> hist;
    const size_t n = p->dim();
    cudaStream_t st = p->ctx->stream;
    if (where == FPC_DEVICE) {
      check_dev_aligned(b, "fpc_gmres");
      check_dev_aligned(x, "fpc_gmres");
      gmres_dev(pl, b, x, cfg, rep, hist);
    } else {
      ensure_staging(p);
      upload(p->d_in, b, n * sizeof(double), st);
      try {
        gmres_dev(pl, p->d_in, p->d_out, cfg, rep, hist, x);
      } catch (...) {
        if (p->ctx->aux) cudaStreamSynchronize(p->ctx->aux);
        throw;
      }
      ck(cudaStreamSynchronize(st), "sync");
      ck(cudaStreamSynchronize(p->ctx->aux), "sync");
    }
    rep->iterations_exact = rep->iterations;
    rep->history_len = int(hist.size());
    for (int i = 0; i < int(hist.size()) && i < history_cap; ++i) history[i] = hist[size_t(i)];
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---------------------------------------------------------------------------- BiCGSTAB
// bicgstab_left (krylov.hpp:204-280) on the device: the recurrence on preconditioned vectors with
// the true residual carried alongside from the same matvec outputs.  Scalars go to the host at
// three sync points per iteration (the half-step test, omega, the full-step test); alpha is formed
// on the device from rho and the denominator so the s update needs no extra round trip.
static void bicgstab_dev(fpc_plan_s* pl, const double* b, double* x, const fpc_solver_config& cfg,
                         fpc_report* rep, std::vector<double>& hist, double* host_x = nullptr, bool* copied = nullptr) {
  fpc_problem_s* p = pl->prob;
  fpc_context_s* c = p->ctx;
  const size_t n = p->dim();
  cudaStream_t st = c->stream;
  GmresState S{pl, c, n, st, {}, 0};
  ck(cudaMemsetAsync(x, 0, n * sizeof(double), st), "memset");
  dots_into(S, {}, 0, b, true, 0);
  ck(cudaMemcpyAsync(c->hpin, c->dscal, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  const double norm_b = std::sqrt(c->hpin[0]);
  rep->iterations_exact = 0.0;
  if (norm_b == 0.0) {
    rep->converged = 1;
    return;
  }
  constexpr double kFloor = 1e-300;  // krylov.hpp:215
  // workspace in the plan's basis slots: r (= s), r_true (= s_true), rhat, p, q (= t_orig), v, t
  double* r = basis_buf(pl, 0, n);
  double* rt = basis_buf(pl, 1, n);
  double* rhat = basis_buf(pl, 2, n);
  double* pv = basis_buf(pl, 3, n);
  double* q = basis_buf(pl, 4, n);
  double* v = basis_buf(pl, 5, n);
  double* t = basis_buf(pl, 6, n);
  // device scalar slots: [kR] rho, [kD] denom (adjacent: k_bicg_s reads both), [kS] ||s_true||^2,
  // [kT] <s,t>, ||t||^2, [kN] ||r_true||^2, next rho
  constexpr int kR = 1100, kD = 1101, kS = 1104, kT = 1108, kN = 1112;
  const int stride = fpc_context_s::kPartialStride;
  ck(cudaMemcpyAsync(rt, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
  pc_apply_dev(pl, b, r, 1.0);
  ck(cudaMemcpyAsync(rhat, r, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
  dots_into(S, {}, 0, r, true, kR);  // rho_0 = <rhat, r> = ||r||^2
  ck(cudaMemcpyAsync(c->hpin + kR, c->dscal + kR, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  double rho = c->hpin[kR], rho_prev = 1.0, alpha = 1.0, omega = 1.0;
  for (int k = 0; k < cfg.max_iter; ++k) {
    if (std::abs(rho) < kFloor) break;
    const double beta = k == 0 ? 0.0 : (rho / rho_prev) * (alpha / omega);
    LAUNCH("bicg_p", st, fpc::launch_bicg_p(r, v, pv, beta, omega, n, k == 0, st));
    matvec_dev(p, pv, q);
    pc_apply_dev(pl, q, v, 1.0);
    fpc::VecSet vs{};
    vs.v[0] = rhat;
    vs.s[0] = 1.0;
    LAUNCH("dots", st, fpc::launch_dots(vs, 1, v, n, c->partial, stride, 0, false, st));
    LAUNCH("reduce", st, fpc::launch_reduce(c->partial, stride, 1, c->dscal + kD, false, st));
    LAUNCH("bicg_s", st, fpc::launch_bicg_s(r, rt, v, q, c->dscal + kR, n, c->partial, st));
    LAUNCH("reduce", st, fpc::launch_reduce(c->partial, 1, 1, c->dscal + kS, false, st));
    ck(cudaMemcpyAsync(c->hpin + kD, c->dscal + kD, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(c->hpin + kS, c->dscal + kS, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    const double denom = c->hpin[kD];
    if (std::abs(denom) < kFloor) break;
    alpha = rho / denom;
    const double rel_half = std::sqrt(c->hpin[kS]) / norm_b;
    hist.push_back(rel_half);
    if (rel_half <= cfg.tol) {
      LAUNCH("axpy", st, fpc::launch_axpy(alpha, pv, x, n, st));
      rep->iterations_exact = k + 0.5;
      rep->converged = 1;
      rep->final_relative_residual = rel_half;
      break;
    }
    matvec_dev(p, r, q);  // t_orig = A s (s lives in r; t_orig over q)
    pc_apply_dev(pl, q, t, 1.0);
    vs.v[0] = r;  // <s, t> and ||t||^2
    LAUNCH("dots", st, fpc::launch_dots(vs, 1, t, n, c->partial, stride, 0, true, st));
    LAUNCH("reduce", st, fpc::launch_reduce(c->partial, stride, 2, c->dscal + kT, false, st));
    ck(cudaMemcpyAsync(c->hpin + kT, c->dscal + kT, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    const double tt = c->hpin[kT + 1];
    if (tt < kFloor) break;
    omega = c->hpin[kT] / tt;
    LAUNCH("bicg_x", st, fpc::launch_bicg_x(x, pv, r, t, rt, q, rhat, alpha, omega, n, c->partial, st));
    LAUNCH("reduce", st, fpc::launch_reduce(c->partial, 2, 2, c->dscal + kN, false, st));
    ck(cudaMemcpyAsync(c->hpin + kN, c->dscal + kN, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    const double rel = std::sqrt(c->hpin[kN]) / norm_b;
    hist.push_back(rel);
    rep->iterations_exact = k + 1.0;
    rep->final_relative_residual = rel;
    if (rel <= cfg.tol) {
      rep->converged = 1;
      break;
    }
    if (std::abs(omega) < kFloor) break;
    rho_prev = rho;
    rho = c->hpin[kN + 1];
    ck(cudaMemcpyAsync(c->dscal + kR, c->dscal + kN + 1, sizeof(double), cudaMemcpyDeviceToDevice, st), "rho");
  }
  if (host_x) {  // x is final: copy it back under the true-residual check (as gmres_dev)
    copy_out_async(c, host_x, x, pl->prob->dim());
    *copied = true;
  }
  rep->true_relative_residual = resid_norm_dev(pl, b, x) / norm_b;
}

int fpc_bicgstab(fpc_plan_t pl, const double* b, double* x, const fpc_solver_config* cfg_in,
                 fpc_report* rep, double* history, int history_cap, int where) {
  if (!pl || !rep) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    check_ptr(b, "fpc_bicgstab");
    check_ptr(x, "fpc_bicgstab");
    fpc_solver_config cfg{1e-9, 200, 0, FPC_SWEEP_HALF};
    if (cfg_in) cfg = *cfg_in;
    if (cfg.sweep != FPC_SWEEP_HALF && cfg.sweep != FPC_SWEEP_FULL) throw InvalidArg{"fpc_bicgstab: bad sweep"};
    pl->sweep_mode = cfg.sweep;
    fpc_problem_s* p = pl->prob;
    DeviceGuard g(p->ctx->device);
    const auto t0 = std::chrono::steady_clock::now();
    std::memset(rep, 0, sizeof *rep);
    std::vector<double> hist;
    const size_t n = p->dim();
    cudaStream_t st = p->ctx->stream;
    if (where == FPC_DEVICE) {
      check_dev_aligned(b, "fpc_bicgstab");
      check_dev_aligned(x, "fpc_bicgstab");
      bicgstab_dev(pl, b, x, cfg, rep, hist);
    } else {
      ensure_staging(p);
      upload(p->d_in, b, n * sizeof(double), st);
      bool copied = false;
      try {
        bicgstab_dev(pl, p->d_in, p->d_out, cfg, rep, hist, x, &copied);
      } catch (...) {
        if (p->ctx->aux) cudaStreamSynchronize(p->ctx->aux);
        throw;
      }
      if (!copied) ck(cudaMemcpyAsync(x, p->d_out, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      if (copied) ck(cudaStreamSynchronize(p->ctx->aux), "sync");
    }
    rep->iterations = int(rep->iterations_exact);
    rep->history_len = int(hist.size());
    for (int i = 0; i < int(hist.size()) && i < history_cap; ++i) history[i] = hist[size_t(i)];
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---------------------------------------------------------------------------- shard level
// The per-rank pieces of the frequency-sharded multi-GPU solve (paper_2003_07020_b200/
// distributed.py): device pointers on the context device, stream-ordered on its stream.

int fpc_shard_matvec(fpc_problem_t p, const double* v, double* y, int nt_local, int k_offset) {
  if (!p) return set_err(FPC_INVALID_ARGUMENT, "null problem");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_prob(p->mu);
    check_ptr(v, "fpc_shard_matvec");
    check_ptr(y, "fpc_shard_matvec");
    if (nt_local < 1 || k_offset < 0 || k_offset + nt_local > p->nt)
      throw InvalidArg{"fpc_shard_matvec: bad time range"};
    DeviceGuard g(p->ctx->device);
    cudaStream_t st = p->ctx->stream;
    if (!p->two_dim)
      LAUNCH("matvec_1d", st, fpc::launch_matvec_1d(v, y, p->ns, nt_local, p->log_m, p->d_eig, p->ctx->tw, st, k_offset));
    else
      LAUNCH("matvec_2d", st, fpc::launch_matvec_2d(v, y, p->n, nt_local, p->log_m, p->d_eig, p->d_eig_x, p->ctx->tw, st, k_offset));
  });
}

int fpc_shard_time_fwd(fpc_plan_t pl, const double* v, double* Z, int ns_local, double s_in) {
  if (!pl) return set_err(FPC_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    fpc_problem_s* p = pl->prob;
    if (p->generic) throw Unsupported{"fpc_shard_time_fwd: power-of-two sizes only (the sharded path)"};
    if (ns_local < 1 || ns_local > p->ns) throw InvalidArg{"fpc_shard_time_fwd: bad column count"};
    DeviceGuard g(p->ctx->device);
    cudaStream_t st = p->ctx->stream;
    LAUNCH("time_fwd", st, fpc::launch_time_fwd(v, reinterpret_cast<double2*>(Z), ns_local, p->nt, pl->d_sf, s_in, p->ctx->tw, st));
  });
}

int fpc_shard_tau(fpc_plan_t pl, double* Z, int row0, int nrows, int forward) {
  if (!pl) return set_err(FPC_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    fpc_problem_s* p = pl->prob;
    if (p->generic) throw Unsupported{"fpc_shard_tau: power-of-two sizes only (the sharded path)"};
    if (row0 < 0 || nrows < 0 || row0 + nrows > pl->solve_count)
      throw InvalidArg{"fpc_shard_tau: bad frequency range"};
    if (nrows == 0) return;
    DeviceGuard g(p->ctx->device);
    cudaStream_t st = p->ctx->stream;
    double2* z = reinterpret_cast<double2*>(Z);
    if (!p->two_dim)
      LAUNCH("tau_solve_1d", st, fpc::launch_tau_solve_1d(z, p->ns, nrows, pl->d_lambda + row0, pl->d_sigma, p->dt, p->ctx->tw, st, forward != 0));
    else
      LAUNCH("tau_solve_2d", st, fpc::launch_tau_solve_2d(z, p->n, nrows, pl->d_lambda + row0, pl->d_sigma, p->dt, p->ctx->tw, st, forward != 0));
  });
}

int fpc_shard_time_inv(fpc_plan_t pl, const double* Z, double* z, int ns_local) {
  if (!pl) return set_err(FPC_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    fpc_problem_s* p = pl->prob;
    if (p->generic) throw Unsupported{"fpc_shard_time_inv: power-of-two sizes only (the sharded path)"};
    if (ns_local < 1 || ns_local > p->ns) throw InvalidArg{"fpc_shard_time_inv: bad column count"};
    DeviceGuard g(p->ctx->device);
    cudaStream_t st = p->ctx->stream;
    LAUNCH("time_inv", st, fpc::launch_time_inv(reinterpret_cast<const double2*>(Z), z, ns_local, p->nt, pl->d_sb, p->ctx->tw, st));
  });
}

static void check_commuted_shard(const fpc_problem_s* p, const char* who) {
  if (p->generic) throw Unsupported{std::string(who) + ": power-of-two sizes only"};
}

int fpc_shard_dst_levels(fpc_plan_t pl, const double* v, double* out, int nt_local, double s_in) {
  if (!pl || !v || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    fpc_problem_s* p = pl->prob;
    check_commuted_shard(p, "fpc_shard_dst_levels");
    if (nt_local < 2 || nt_local % 2 || nt_local > p->nt)
      throw InvalidArg{"fpc_shard_dst_levels: nt_local must be even and <= n_time"};
    if (v == out) throw InvalidArg{"fpc_shard_dst_levels: input and output must be disjoint"};
    DeviceGuard g(p->ctx->device);
    cudaStream_t st = p->ctx->stream;
    // any pairing of levels into complex rows is valid (the transform is per level)
    dst_levels_dev(pl, v, out, nt_local, s_in);
  });
}

int fpc_shard_time_solve(fpc_plan_t pl, const double* u, double* z, int col0, int ns_local, int forward) {
  if (!pl || !u || !z) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk_plan(pl->mu);
    std::lock_guard<std::recursive_mutex> lk_prob(pl->prob->mu);
    fpc_problem_s* p = pl->prob;
    check_commuted_shard(p, "fpc_shard_time_solve");
    if (col0 < 0 || ns_local < 1 || col0 + ns_local > p->ns) throw InvalidArg{"fpc_shard_time_solve: bad column range"};
    DeviceGuard g(p->ctx->device);
    cudaStream_t st = p->ctx->stream;
    LAUNCH("time_solve", st,
           fpc::launch_time_solve(u, z, ns_local, p->nt, pl->d_sf, pl->d_sb, 1.0, pl->d_lambda, pl->d_sigma + col0,
                                  p->dt, p->ctx->tw, st, forward != 0));
  });
}

// out_host[i] = s_i <V_i, w> (i < nv), out_host[nv] = <w, w> when with_norm; synchronous.
int fpc_shard_dots(fpc_context_t c, const double* const* V, const double* scales, int nv,
                   const double* w, size_t n, int with_norm, double* out_host) {
  if (!c || !out_host) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (nv < 0 || nv > 250) throw InvalidArg{"fpc_shard_dots: 0 <= nv <= 250"};
    for (int i = 0; i < nv; ++i) check_dev_aligned(V[i], "fpc_shard_dots");
    check_dev_aligned(w, "fpc_shard_dots");
    DeviceGuard g(c->device);
    GmresState S{nullptr, c, n, c->stream, std::vector<double>(scales, scales + nv), 0};
    std::vector<const double*> vv(V, V + nv);
    dots_into(S, vv, nv, w, nv == 0 ? true : with_norm != 0, 0);
    const int cnt = nv + ((with_norm || nv == 0) ? 1 : 0);
    ck(cudaMemcpyAsync(c->hpin, c->dscal, size_t(cnt) * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    std::memcpy(out_host, c->hpin, size_t(cnt) * sizeof(double));
  });
}

// ---------------------------------------------------------------------------- peer-store transport
int fpc_ipc_get_handle(const void* dptr, void* handle64) {
  if (!dptr || !handle64) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)), "cudaIpcGetMemHandle");
    std::memcpy(handle64, &h, sizeof h);
  });
}

int fpc_ipc_open(fpc_context_t c, const void* handle64, void** dptr) {
  if (!c || !handle64 || !dptr) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    ck(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

int fpc_ipc_close(fpc_context_t c, void* dptr) {
  if (!c || !dptr) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    DeviceGuard g(c->device);
    ck(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle");
  });
}

int fpc_shard_scatter_p2p(fpc_context_t c, const double* src, int rows, int cols, int es, int split_cols,
                          double* const* dst, const int* off, const int* stride, int nranks, int row_base,
                          int col_base) {
  if (!c || !dst || !off || !stride) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (nranks < 1 || nranks > fpc::kP2PMaxRanks) throw InvalidArg{"fpc_shard_scatter_p2p: 1 <= nranks <= 8"};
    if (es != 1 && es != 2) throw InvalidArg{"fpc_shard_scatter_p2p: es must be 1 or 2"};
    if (rows < 0 || cols < 0 || row_base < 0 || col_base < 0) throw InvalidArg{"fpc_shard_scatter_p2p: negative size"};
    if (size_t(rows) * size_t(cols) > 0) check_ptr(src, "fpc_shard_scatter_p2p");
    fpc::P2PScatter a{};
    for (int d = 0; d < nranks; ++d) {
      check_ptr(dst[d], "fpc_shard_scatter_p2p");
      if (es == 2) check_dev_aligned(dst[d], "fpc_shard_scatter_p2p");
      if (d > 0 && off[d] < off[d - 1]) throw InvalidArg{"fpc_shard_scatter_p2p: offsets must be non-decreasing"};
      if (stride[d] < 0) throw InvalidArg{"fpc_shard_scatter_p2p: negative stride"};
      a.dst[d] = dst[d];
      a.off[d] = off[d];
      a.stride[d] = stride[d];
    }
    if (off[0] != 0) throw InvalidArg{"fpc_shard_scatter_p2p: off[0] must be 0"};
    if (es == 2) check_dev_aligned(src, "fpc_shard_scatter_p2p");
    DeviceGuard g(c->device);
    LAUNCH("scatter_p2p", c->stream, fpc::launch_p2p_scatter(src, rows, cols, es, split_cols != 0, a, nranks,
                                                               row_base, col_base, c->stream));
  });
}

// The same dots left on the device: out_dev[0..cnt) (device pointer), stream-ordered, no host sync
// -- the sharded solver all-reduces them in place with NCCL and reads the sum once.
int fpc_shard_dots_dev(fpc_context_t c, const double* const* V, const double* scales, int nv, const double* w,
                       size_t n, int with_norm, double* out_dev) {
  if (!c || !out_dev) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (nv < 0 || nv > 250) throw InvalidArg{"fpc_shard_dots_dev: 0 <= nv <= 250"};
    for (int i = 0; i < nv; ++i) check_dev_aligned(V[i], "fpc_shard_dots_dev");
    check_dev_aligned(w, "fpc_shard_dots_dev");
    DeviceGuard g(c->device);
    GmresState S{nullptr, c, n, c->stream, std::vector<double>(scales, scales + nv), 0};
    std::vector<const double*> vv(V, V + nv);
    dots_into(S, vv, nv, w, nv == 0 ? true : with_norm != 0, 0);
    const int cnt = nv + ((with_norm || nv == 0) ? 1 : 0);
    ck(cudaMemcpyAsync(out_dev, c->dscal, size_t(cnt) * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
  });
}

// w <- w - sum_i coef_i V_i with ||w||^2 left at norm2_dev (device pointer), no host sync
int fpc_shard_update_dev(fpc_context_t c, const double* const* V, const double* coef, int nv, double* w, size_t n,
                         double* norm2_dev) {
  if (!c || !norm2_dev) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (nv < 0 || nv > 250) throw InvalidArg{"fpc_shard_update_dev: 0 <= nv <= 250"};
    for (int i = 0; i < nv; ++i) check_dev_aligned(V[i], "fpc_shard_update_dev");
    check_dev_aligned(w, "fpc_shard_update_dev");
    DeviceGuard g(c->device);
    std::vector<double> ones(size_t(nv), 1.0);
    // the coefficient and pointer tables go through pinned staging (hpin), so the copies are
    // genuinely asynchronous: wait for the previous user of that staging area first
    ck(cudaStreamSynchronize(c->stream), "sync");
    std::memcpy(c->hpin + 700, coef, size_t(nv) * sizeof(double));
    std::memcpy(c->hpin + 1300, ones.data(), size_t(nv) * sizeof(double));
    ck(cudaMemcpyAsync(c->dvptr, V, size_t(nv) * sizeof(double*), cudaMemcpyHostToDevice, c->stream), "vptr");
    ck(cudaMemcpyAsync(c->dscales, c->hpin + 1300, size_t(nv) * sizeof(double), cudaMemcpyHostToDevice, c->stream),
       "scales");
    ck(cudaMemcpyAsync(c->dscal + 700, c->hpin + 700, size_t(nv) * sizeof(double), cudaMemcpyHostToDevice, c->stream),
       "coef");
    LAUNCH("update", c->stream, fpc::launch_update(c->dvptr, c->dscales, c->dscal + 700, nv, w, n, c->partial, c->stream));
    LAUNCH("reduce", c->stream, fpc::launch_reduce(c->partial, 1, 1, norm2_dev, false, c->stream));
  });
}

// w <- w - sum_i coef_i * V_i (coef on the host, scales already folded in); returns ||w||^2.
int fpc_shard_update(fpc_context_t c, const double* const* V, const double* coef, int nv, double* w,
                     size_t n, double* norm2_host) {
  if (!c || !norm2_host) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (nv < 0 || nv > 250) throw InvalidArg{"fpc_shard_update: 0 <= nv <= 250"};
    for (int i = 0; i < nv; ++i) check_dev_aligned(V[i], "fpc_shard_update");
    check_dev_aligned(w, "fpc_shard_update");
    DeviceGuard g(c->device);
    std::vector<double> ones(size_t(nv), 1.0);
    ck(cudaMemcpyAsync(c->dvptr, V, size_t(nv) * sizeof(double*), cudaMemcpyHostToDevice, c->stream), "vptr");
    ck(cudaMemcpyAsync(c->dscales, ones.data(), size_t(nv) * sizeof(double), cudaMemcpyHostToDevice, c->stream), "scales");
    std::memcpy(c->hpin + 700, coef, size_t(nv) * sizeof(double));
    ck(cudaMemcpyAsync(c->dscal + 700, c->hpin + 700, size_t(nv) * sizeof(double), cudaMemcpyHostToDevice, c->stream), "coef");
    LAUNCH("update", c->stream, fpc::launch_update(c->dvptr, c->dscales, c->dscal + 700, nv, w, n, c->partial, c->stream));
    LAUNCH("reduce", c->stream, fpc::launch_reduce(c->partial, 1, 1, c->dscal + 512, false, c->stream));
    ck(cudaMemcpyAsync(c->hpin + 512, c->dscal + 512, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    *norm2_host = c->hpin[512];
  });
}

// u = sum_i coef_i V_i (coef on the host)
int fpc_shard_lincomb(fpc_context_t c, const double* const* V, const double* coef, int nv, double* u,
                      size_t n) {
  if (!c) return set_err(FPC_INVALID_ARGUMENT, "null context");
  return guarded([&] {
    if (nv < 1 || nv > 250) throw InvalidArg{"fpc_shard_lincomb: 1 <= nv <= 250"};
    for (int i = 0; i < nv; ++i) check_dev_aligned(V[i], "fpc_shard_lincomb");
    check_dev_aligned(u, "fpc_shard_lincomb");
    DeviceGuard g(c->device);
    std::vector<double> ones(size_t(nv), 1.0);
    ck(cudaMemcpyAsync(c->dvptr, V, size_t(nv) * sizeof(double*), cudaMemcpyHostToDevice, c->stream), "vptr");
    ck(cudaMemcpyAsync(c->dscales, ones.data(), size_t(nv) * sizeof(double), cudaMemcpyHostToDevice, c->stream), "scales");
    std::memcpy(c->hpin + 700, coef, size_t(nv) * sizeof(double));
    ck(cudaMemcpyAsync(c->dscal + 700, c->hpin + 700, size_t(nv) * sizeof(double), cudaMemcpyHostToDevice, c->stream), "coef");
    LAUNCH("lincomb", c->stream, fpc::launch_lincomb(c->dvptr, c->dscales, c->dscal + 700, nv, u, n, c->stream));
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

// ---------------------------------------------------------------------------- generic GMRES
// gmres_right(n, apply_a, apply_pinv, b, cfg) for arbitrary HOST callables (krylov.hpp:83-192):
// the reference's iteration -- Gram-Schmidt with its conditional re-orthogonalisation (threshold
// 1/sqrt(2), krylov.hpp:107, 123-130), Givens rotations (133-151), the |g_{j+1}|/||b|| stop test
// (154-159), the breakdown test (160-165), x = P^{-1}(sum y_k v_k) (180-183) and the fresh TRR
// (188) -- with the Krylov basis resident on the device and the dots / updates / combinations run
// by the library's deterministic vector kernels.  Each step stages v_j to the host once, calls
// apply_pinv then apply_a there (z never leaves the host) and uploads w.  restart = m > 0: the
// GMRES(m) emulation of SURVEY §8(c) (x0 = 0 per cycle on the residual).
namespace {
struct HostPinned {
  double* p = nullptr;
  explicit HostPinned(size_t n) { ck(cudaMallocHost(&p, std::max<size_t>(n, 1) * sizeof(double)), "cudaMallocHost"); }
  ~HostPinned() { if (p) cudaFreeHost(p); }
};
struct DevVec {
  double* p = nullptr;
  explicit DevVec(size_t n) { p = dalloc<double>(n + 2); }
  ~DevVec() { if (p) cudaFree(p); }
  DevVec(DevVec&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevVec(const DevVec&) = delete;
};
void call_op(fpc_apply_fn f, void* user, const double* in, double* out, size_t n, const char* who) {
  const int rc = f(in, out, n, user);
  if (rc != 0) throw RuntimeErr{std::string(who) + ": the callable reported failure (status " + std::to_string(rc) + ")"};
}
}  // namespace

int fpc_gmres_callbacks(fpc_context_t c, size_t n, fpc_apply_fn apply_a, void* a_user, fpc_apply_fn apply_pinv,
                        void* p_user, const double* b, double* x, const fpc_solver_config* cfg_in, fpc_report* report,
                        double* history, int history_cap) {
  if (!c || !apply_a || !apply_pinv || !b || !x || !cfg_in || !report)
    return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    const fpc_solver_config cfg = *cfg_in;
    if (n == 0) throw InvalidArg{"gmres_right: empty system"};
    if (cfg.max_iter < 0) throw InvalidArg{"gmres_right: max_iter must be non-negative"};
    const int mcyc = (cfg.restart > 0 && cfg.restart < cfg.max_iter) ? cfg.restart : cfg.max_iter;
    if (mcyc + 1 > 250) throw Unsupported{"gmres_right (callables): at most 249 steps per cycle"};
    DeviceGuard g(c->device);
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t st = c->stream;
    *report = fpc_report{};
    HostPinned hin(n), hout(n), hz(n);
    DevVec dr(n), dw(n);
    std::vector<DevVec> V;
    V.reserve(size_t(mcyc) + 1);
    auto h2d = [&](double* d, const double* h) {
      ck(cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
    };
    auto d2h = [&](double* h, const double* d) {
      ck(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
    };
    auto check_rc = [](int rc) {
      if (rc != FPC_OK) throw RuntimeErr{g_err};
    };
    auto norm2 = [&](const double* d) {
      double out = 0.0;
      check_rc(fpc_shard_dots(c, nullptr, nullptr, 0, d, n, 1, &out));
      return std::sqrt(out);
    };
    std::vector<double> xh(n, 0.0), bh(b, b + n), rh(bh);
    h2d(dr.p, b);
    const double norm_b = norm2(dr.p);
    int hist_len = 0, total = 0, cycles = 0, reorth = 0;
    bool conv = norm_b == 0.0;
    double last_rel = conv ? 0.0 : 1.0, norm_r = norm_b;
    while (!conv && total < cfg.max_iter) {
      const int budget = std::min(mcyc, cfg.max_iter - total);
      const double tol_c = cfg.tol * norm_b / norm_r;  // the cycle's tolerance relative to ||r||
      // v_0 = r / ||r||
      while (V.size() < size_t(budget) + 1) V.emplace_back(n);
      {
        const double* src[1] = {dr.p};
        const double coef[1] = {1.0 / norm_r};
        check_rc(fpc_shard_lincomb(c, src, coef, 1, V[0].p, n));
      }
      std::vector<std::vector<double>> H;
      std::vector<double> gc, gs, gg{norm_r};
      int steps = 0;
      bool inner_conv = false;
      for (int j = 0; j < budget; ++j) {
        d2h(hin.p, V[size_t(j)].p);
        call_op(apply_pinv, p_user, hin.p, hz.p, n, "apply_pinv");
        call_op(apply_a, a_user, hz.p, hout.p, n, "apply_a");
        h2d(dw.p, hout.p);
        std::vector<const double*> vp(static_cast<size_t>(j) + 1);
        for (int i = 0; i <= j; ++i) vp[size_t(i)] = V[size_t(i)].p;
        std::vector<double> ones(size_t(j) + 1, 1.0), hcol(size_t(j) + 2, 0.0), dd(size_t(j) + 2);
        const double norm_before = norm2(dw.p);
        // one Gram-Schmidt pass (all projections, then the update), repeated once when the norm
        // dropped below 1/sqrt(2) of its value before (krylov.hpp:116-131)
        double norm_w = norm_before;
        for (int pass = 0; pass < 2; ++pass) {
          check_rc(fpc_shard_dots(c, vp.data(), ones.data(), j + 1, dw.p, n, 0, dd.data()));
          double nw2 = 0.0;
          check_rc(fpc_shard_update(c, vp.data(), dd.data(), j + 1, dw.p, n, &nw2));
          for (int i = 0; i <= j; ++i) hcol[size_t(i)] += dd[size_t(i)];
          const double prev = pass == 0 ? norm_before : norm_w;
          norm_w = std::sqrt(std::max(nw2, 0.0));
          if (pass == 0 && !(norm_w < 0.70710678118654752 * prev)) break;
          if (pass == 1) ++reorth;
        }
        hcol[size_t(j) + 1] = norm_w;
        for (int i = 0; i < j; ++i) {  // previous rotations (krylov.hpp:133-140)
          const double hi = hcol[size_t(i)], hi1 = hcol[size_t(i) + 1];
          hcol[size_t(i)] = gc[size_t(i)] * hi + gs[size_t(i)] * hi1;
          hcol[size_t(i) + 1] = -gs[size_t(i)] * hi + gc[size_t(i)] * hi1;
        }
        const double hj = hcol[size_t(j)], hj1 = hcol[size_t(j) + 1];
        const double rad = std::hypot(hj, hj1);
        const double cs = rad > 0.0 ? hj / rad : 1.0, sn = rad > 0.0 ? hj1 / rad : 0.0;
        gc.push_back(cs);
        gs.push_back(sn);
        hcol[size_t(j)] = rad;
        hcol[size_t(j) + 1] = 0.0;
        gg.push_back(-sn * gg[size_t(j)]);
        gg[size_t(j)] *= cs;
        H.push_back(hcol);
        steps = j + 1;
        const double rel_c = std::abs(gg[size_t(j) + 1]) / norm_r;
        last_rel = rel_c * norm_r / norm_b;
        if (history && hist_len < history_cap) history[hist_len] = last_rel;
        ++hist_len;
        if (rel_c <= tol_c) {
          inner_conv = true;
          break;
        }
        if (norm_w <= 1e-14 * std::max(1.0, norm_before)) break;  // breakdown (krylov.hpp:160-165)
        const double* src[1] = {dw.p};
        const double coef[1] = {1.0 / norm_w};
        check_rc(fpc_shard_lincomb(c, src, coef, 1, V[size_t(j) + 1].p, n));
      }
      total += steps;
      ++cycles;
      if (steps > 0) {  // y by back substitution, u = V y, delta = P^{-1} u (krylov.hpp:175-183)
        std::vector<double> y(size_t(steps), 0.0);
        for (int i = steps - 1; i >= 0; --i) {
          double sacc = gg[size_t(i)];
          for (int k = i + 1; k < steps; ++k) sacc -= H[size_t(k)][size_t(i)] * y[size_t(k)];
          y[size_t(i)] = sacc / H[size_t(i)][size_t(i)];
        }
        std::vector<const double*> vp(static_cast<size_t>(steps));
        for (int i = 0; i < steps; ++i) vp[size_t(i)] = V[size_t(i)].p;
        check_rc(fpc_shard_lincomb(c, vp.data(), y.data(), steps, dw.p, n));
        d2h(hin.p, dw.p);
        call_op(apply_pinv, p_user, hin.p, hz.p, n, "apply_pinv");
        for (size_t i = 0; i < n; ++i) xh[i] += hz.p[i];
      }
      if (inner_conv) conv = true;
      if (conv || steps == 0 || total >= cfg.max_iter) break;
      // r = b - A x for the next cycle
      call_op(apply_a, a_user, xh.data(), hout.p, n, "apply_a");
      for (size_t i = 0; i < n; ++i) rh[i] = bh[i] - hout.p[i];
      h2d(dr.p, rh.data());
      norm_r = norm2(dr.p);
      if (norm_r == 0.0) conv = true;
    }
    // fresh true residual (krylov.hpp:188)
    double trr = 0.0;
    if (norm_b > 0.0) {
      call_op(apply_a, a_user, xh.data(), hout.p, n, "apply_a");
      for (size_t i = 0; i < n; ++i) rh[i] = bh[i] - hout.p[i];
      h2d(dr.p, rh.data());
      trr = norm2(dr.p) / norm_b;
    }
    std::copy(xh.begin(), xh.end(), x);
    report->converged = conv ? 1 : 0;
    report->iterations = total;
    report->iterations_exact = double(total);
    report->restarts = cycles > 0 ? cycles - 1 : 0;
    report->reorthogonalizations = reorth;
    report->final_relative_residual = last_rel;
    report->true_relative_residual = trr;
    report->history_len = hist_len;
    report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"

// ============================================================================ multi-device
// One process drives 1..8 devices (SURVEY §8(b) "context over 1..8 devices", §8(e)): the solve of
// the frequency-sharded layout (distributed.py's ShardedSolver, reference ordering) behind the
// C-ABI.  Krylov vectors are time-sharded (rank r owns time levels [r nt_loc, (r+1) nt_loc), stored
// after two halo levels); the matvec takes the BDF2 halo from rank r-1 by a peer copy; the PC apply
// runs the four transpositions time -> space -> frequency -> space -> time as peer-store kernels
// (kernels_p2p.cu: every element stored straight into its slot of the owner's buffer over NVLink),
// each ordered by events (every rank's stream waits for every rank's exchange kernel); the tau solves
// of the retained frequencies (alpha_circulant.hpp:160) are split across the ranks.  The
// Gram-Schmidt dots are per-rank partials summed in rank order on the host (the Hessenberg
// recurrence needs them there anyway; deterministic), the updates and combinations are local.
// Ranks may share a device (devices = {0, 0, ...}): nothing waits on another rank inside a kernel,
// so one GPU runs the G-rank schedule for testing.
struct fpc_multi_s {
  int G = 0;
  std::vector<int> devices;
  std::vector<fpc_context_s*> ctx;
  std::vector<cudaEvent_t> ev;
};

struct fpc_sharded_s {
  fpc_multi_s* m = nullptr;
  int G = 0, nt = 0, ns = 0, n = 0, two_dim = 0, nt_loc = 0, H = 0;
  std::vector<int> cs, co, hs, ho, ts;  // column split of Ns, frequency split of H, time offsets
  std::vector<fpc_problem_s*> prob;
  std::vector<fpc_plan_s*> plan;
  std::vector<double*> cols, rows, zf, zb, zt, tmp;  // exchange buffers per rank
  size_t vec_len = 0;                                  // (nt_loc + 2) * ns per rank (halo first)
};

namespace {
std::vector<int> split_counts(int n, int G) {
  std::vector<int> c(size_t(G), n / G);
  for (int i = 0; i < n % G; ++i) ++c[size_t(i)];
  return c;
}
std::vector<int> offsets_of(const std::vector<int>& c) {
  std::vector<int> o(c.size() + 1, 0);
  for (size_t i = 0; i < c.size(); ++i) o[i + 1] = o[i] + c[i];
  return o;
}
void check_rc(int rc) {
  if (rc != FPC_OK) throw RuntimeErr{g_err};
}

// every rank's stream waits for everything enqueued so far on every rank's stream
void multi_barrier(fpc_multi_s* m) {
  for (int r = 0; r < m->G; ++r) {
    DeviceGuard g(m->devices[size_t(r)]);
    ck(cudaEventRecord(m->ev[size_t(r)], m->ctx[size_t(r)]->stream), "cudaEventRecord");
  }
  for (int r = 0; r < m->G; ++r) {
    DeviceGuard g(m->devices[size_t(r)]);
    for (int q = 0; q < m->G; ++q)
      if (q != r) ck(cudaStreamWaitEvent(m->ctx[size_t(r)]->stream, m->ev[size_t(q)], 0), "cudaStreamWaitEvent");
  }
}

// A sharded vector: one device buffer per rank, the local levels at offset 2 ns (halo first).
struct SVec {
  std::vector<double*> p;
};
double* loc(const fpc_sharded_s* s, const SVec& v, int r) { return v.p[size_t(r)] + 2 * size_t(s->ns); }

SVec svec_alloc(fpc_sharded_s* s) {
  SVec v;
  for (int r = 0; r < s->G; ++r) {
    DeviceGuard g(s->m->devices[size_t(r)]);
    v.p.push_back(dalloc<double>(s->vec_len + 2));
  }
  return v;
}
void svec_free(fpc_sharded_s* s, SVec& v) {
  for (int r = 0; r < s->G && r < int(v.p.size()); ++r) {
    DeviceGuard g(s->m->devices[size_t(r)]);
    cudaFree(v.p[size_t(r)]);
  }
  v.p.clear();
}

void sh_matvec(fpc_sharded_s* s, const SVec& v, SVec& y) {
  const size_t ns = size_t(s->ns), nl = size_t(s->nt_loc);
  multi_barrier(s->m);
  for (int r = 1; r < s->G; ++r) {  // BDF2 halo: the two last levels of rank r-1
    DeviceGuard g(s->m->devices[size_t(r)]);
    ck(cudaMemcpyPeerAsync(v.p[size_t(r)], s->m->devices[size_t(r)], loc(s, v, r - 1) + (nl - 2) * ns,
                           s->m->devices[size_t(r - 1)], 2 * ns * sizeof(double), s->m->ctx[size_t(r)]->stream),
       "halo copy");
  }
  for (int r = 0; r < s->G; ++r)
    check_rc(fpc_shard_matvec(s->prob[size_t(r)], loc(s, v, r), loc(s, y, r), s->nt_loc, s->ts[size_t(r)]));
}

void sh_exchange(fpc_sharded_s* s, const std::vector<const double*>& src, int rows, const std::vector<int>& cols,
                 int es, bool split_cols, const std::vector<double*>& dst, const std::vector<int>& off,
                 const std::vector<int>& stride, const std::vector<int>& row_base, const std::vector<int>& col_base) {
  multi_barrier(s->m);
  for (int r = 0; r < s->G; ++r)
    check_rc(fpc_shard_scatter_p2p(s->m->ctx[size_t(r)], src[size_t(r)], rows, cols[size_t(r)], es, split_cols ? 1 : 0,
                                   dst.data(), off.data(), stride.data(), s->G, row_base[size_t(r)], col_base[size_t(r)]));
  multi_barrier(s->m);
}

// z = P^{-1} (s_in v), reference ordering (alpha_circulant.hpp:137-199), four peer-store exchanges
void sh_pc_apply(fpc_sharded_s* s, const SVec& v, SVec& z, double s_in) {
  const int G = s->G, ns = s->ns;
  std::vector<const double*> src(static_cast<size_t>(G));
  std::vector<int> colsz(static_cast<size_t>(G)), rb(static_cast<size_t>(G)), cb(static_cast<size_t>(G), 0);
  // 1. time -> space: rank r's [nt_loc][ns] levels -> cols[d] [nt][cs_d] rows r nt_loc..
  for (int r = 0; r < G; ++r) {
    src[size_t(r)] = loc(s, v, r);
    colsz[size_t(r)] = ns;
    rb[size_t(r)] = s->ts[size_t(r)];
  }
  std::vector<int> off(s->co.begin(), s->co.end() - 1), stride(s->cs.begin(), s->cs.end());
  sh_exchange(s, src, s->nt_loc, colsz, 1, true, s->cols, off, stride, rb, cb);
  // 2. time FFT on my columns -> zf [H][cs_d] complex
  for (int d = 0; d < G; ++d)
    check_rc(fpc_shard_time_fwd(s->plan[size_t(d)], s->cols[size_t(d)], s->zf[size_t(d)], s->cs[size_t(d)], s_in));
  // 3. space -> frequency: zf[d] rows split by ho -> rows[e] [hs_e][ns] at column co[d]
  for (int d = 0; d < G; ++d) {
    src[size_t(d)] = s->zf[size_t(d)];
    colsz[size_t(d)] = s->cs[size_t(d)];
    rb[size_t(d)] = 0;
    cb[size_t(d)] = s->co[size_t(d)];
  }
  std::vector<int> hoff(s->ho.begin(), s->ho.end() - 1), nsstride(static_cast<size_t>(G), ns);
  sh_exchange(s, src, s->H, colsz, 2, false, s->rows, hoff, nsstride, rb, cb);
  // 4. tau solves of my frequencies
  for (int e = 0; e < G; ++e)
    check_rc(fpc_shard_tau(s->plan[size_t(e)], s->rows[size_t(e)], s->ho[size_t(e)], s->hs[size_t(e)], 0));
  // 5. frequency -> space: rows[e] [hs_e][ns] columns split by co -> zb[d] [H][cs_d] at row ho[e]
  for (int e = 0; e < G; ++e) {
    src[size_t(e)] = s->rows[size_t(e)];
    colsz[size_t(e)] = ns;
    rb[size_t(e)] = s->ho[size_t(e)];
    cb[size_t(e)] = 0;
  }
  // per-source row counts differ (hs_e): exchange rank by rank through the same ordering
  multi_barrier(s->m);
  for (int e = 0; e < G; ++e)
    check_rc(fpc_shard_scatter_p2p(s->m->ctx[size_t(e)], src[size_t(e)], s->hs[size_t(e)], ns, 2, 1, s->zb.data(),
                                   off.data(), stride.data(), G, rb[size_t(e)], 0));
  multi_barrier(s->m);
  // 6. inverse time FFT -> zt [nt][cs_d]
  for (int d = 0; d < G; ++d)
    check_rc(fpc_shard_time_inv(s->plan[size_t(d)], s->zb[size_t(d)], s->zt[size_t(d)], s->cs[size_t(d)]));
  // 7. space -> time: zt[d] rows split by time blocks -> z's local levels of rank r at column co[d]
  std::vector<double*> zdst(static_cast<size_t>(G));
  std::vector<int> toff(static_cast<size_t>(G)), tstride(static_cast<size_t>(G), ns);
  for (int r = 0; r < G; ++r) {
    zdst[size_t(r)] = loc(s, z, r);
    toff[size_t(r)] = s->ts[size_t(r)];
  }
  for (int d = 0; d < G; ++d) {
    src[size_t(d)] = s->zt[size_t(d)];
    colsz[size_t(d)] = s->cs[size_t(d)];
    rb[size_t(d)] = 0;
    cb[size_t(d)] = s->co[size_t(d)];
  }
  sh_exchange(s, src, s->nt, colsz, 1, false, zdst, toff, tstride, rb, cb);
}

// per-rank partial dots <V_i, w> (and ||w||^2), summed over ranks in rank order on the host
std::vector<double> sh_dots(fpc_sharded_s* s, const std::vector<SVec*>& V, const SVec& w, bool with_norm) {
  const int nv = int(V.size());
  const size_t n = size_t(s->nt_loc) * size_t(s->ns);
  const int cnt = nv + (with_norm || nv == 0 ? 1 : 0);
  for (int r = 0; r < s->G; ++r) {
    fpc_context_s* c = s->m->ctx[size_t(r)];
    DeviceGuard g(c->device);
    GmresState S{nullptr, c, n, c->stream, std::vector<double>(size_t(nv), 1.0), 0};
    std::vector<const double*> vv;
    for (auto* x : V) vv.push_back(loc(s, *x, r));
    dots_into(S, vv, nv, loc(s, w, r), nv == 0 ? true : with_norm, 0);
    ck(cudaMemcpyAsync(c->hpin, c->dscal, size_t(cnt) * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  }
  std::vector<double> out(size_t(cnt), 0.0);
  for (int r = 0; r < s->G; ++r) {
    fpc_context_s* c = s->m->ctx[size_t(r)];
    DeviceGuard g(c->device);
    ck(cudaStreamSynchronize(c->stream), "sync");
    for (int i = 0; i < cnt; ++i) out[size_t(i)] += c->hpin[i];
  }
  return out;
}

// w -= sum_i coef_i V_i on every rank; returns ||w||^2
double sh_update(fpc_sharded_s* s, const std::vector<SVec*>& V, const std::vector<double>& coef, SVec& w) {
  double tot = 0.0;
  const size_t n = size_t(s->nt_loc) * size_t(s->ns);
  std::vector<double> part(static_cast<size_t>(s->G));
  for (int r = 0; r < s->G; ++r) {
    std::vector<const double*> vv;
    for (auto* x : V) vv.push_back(loc(s, *x, r));
    check_rc(fpc_shard_update(s->m->ctx[size_t(r)], vv.data(), coef.data(), int(V.size()), loc(s, w, r), n,
                              &part[size_t(r)]));
  }
  for (double p : part) tot += p;
  return tot;
}

void sh_lincomb(fpc_sharded_s* s, const std::vector<SVec*>& V, const std::vector<double>& coef, SVec& u) {
  const size_t n = size_t(s->nt_loc) * size_t(s->ns);
  for (int r = 0; r < s->G; ++r) {
    std::vector<const double*> vv;
    for (auto* x : V) vv.push_back(loc(s, *x, r));
    check_rc(fpc_shard_lincomb(s->m->ctx[size_t(r)], vv.data(), coef.data(), int(V.size()), loc(s, u, r), n));
  }
}

void sh_upload(fpc_sharded_s* s, const double* host, SVec& v) {
  const size_t per = size_t(s->nt_loc) * size_t(s->ns);
  for (int r = 0; r < s->G; ++r) {
    fpc_context_s* c = s->m->ctx[size_t(r)];
    DeviceGuard g(c->device);
    ck(cudaMemcpyAsync(loc(s, v, r), host + size_t(r) * per, per * sizeof(double), cudaMemcpyHostToDevice, c->stream),
       "H2D");
  }
}
void sh_download(fpc_sharded_s* s, const SVec& v, double* host) {
  const size_t per = size_t(s->nt_loc) * size_t(s->ns);
  for (int r = 0; r < s->G; ++r) {
    fpc_context_s* c = s->m->ctx[size_t(r)];
    DeviceGuard g(c->device);
    ck(cudaMemcpyAsync(host + size_t(r) * per, loc(s, v, r), per * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
       "D2H");
  }
  for (int r = 0; r < s->G; ++r) {
    DeviceGuard g(s->m->devices[size_t(r)]);
    ck(cudaStreamSynchronize(s->m->ctx[size_t(r)]->stream), "sync");
  }
}
}  // namespace

extern "C" {

int fpc_multi_create(const int* devices, int n_ranks, fpc_multi_t* out) {
  if (!devices || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (n_ranks < 1 || n_ranks > fpc::kP2PMaxRanks) throw InvalidArg{"fpc_multi_create: 1 <= n_ranks <= 8"};
    auto* m = new fpc_multi_s();
    try {
      m->G = n_ranks;
      m->devices.assign(devices, devices + n_ranks);
      for (int r = 0; r < n_ranks; ++r) {
        fpc_context_t c = nullptr;
        check_rc(fpc_context_create(devices[r], &c));
        m->ctx.push_back(c);
        DeviceGuard g(devices[r]);
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        m->ev.push_back(e);
      }
      for (int a = 0; a < n_ranks; ++a)  // peer access between distinct devices (NVLink / NVSwitch)
        for (int b = 0; b < n_ranks; ++b) {
          if (devices[a] == devices[b]) continue;
          int can = 0;
          ck(cudaDeviceCanAccessPeer(&can, devices[a], devices[b]), "cudaDeviceCanAccessPeer");
          if (!can) throw Unsupported{"fpc_multi_create: devices without peer access"};
          DeviceGuard g(devices[a]);
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else ck(e, "cudaDeviceEnablePeerAccess");
        }
    } catch (...) {
      for (auto* c : m->ctx) fpc_context_destroy(c);
      delete m;
      throw;
    }
    *out = m;
  });
}

int fpc_multi_destroy(fpc_multi_t m) {
  if (!m) return FPC_OK;
  for (int r = 0; r < m->G; ++r) {
    DeviceGuard g(m->devices[size_t(r)]);
    cudaEventDestroy(m->ev[size_t(r)]);
    fpc_context_destroy(m->ctx[size_t(r)]);
  }
  delete m;
  return FPC_OK;
}

static int sharded_create(fpc_multi_t m, bool two_dim, double gx, double gy, double kx, double ky, double h, int n,
                          int n_time, double dt, double alpha, fpc_sharded_t* out) {
  if (!m || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    auto* s = new fpc_sharded_s();
    try {
      s->m = m;
      s->G = m->G;
      s->two_dim = two_dim ? 1 : 0;
      s->n = n;
      s->nt = n_time;
      s->ns = two_dim ? n * n : n;
      s->H = n_time / 2 + 1;
      if (n_time % s->G) throw InvalidArg{"sharded solve: n_time must be divisible by the number of ranks"};
      s->nt_loc = n_time / s->G;
      if (s->G > 1 && s->nt_loc < 2) throw InvalidArg{"sharded solve: at least two time levels per rank"};
      if (s->ns < s->G || s->H < s->G) throw InvalidArg{"sharded solve: fewer columns or frequencies than ranks"};
      s->cs = split_counts(s->ns, s->G);
      s->co = offsets_of(s->cs);
      s->hs = split_counts(s->H, s->G);
      s->ho = offsets_of(s->hs);
      for (int r = 0; r < s->G; ++r) s->ts.push_back(r * s->nt_loc);
      s->vec_len = size_t(s->nt_loc + 2) * size_t(s->ns);
      for (int r = 0; r < s->G; ++r) {
        fpc_problem_t p = nullptr;
        if (two_dim)
          check_rc(fpc_problem_create_2d(m->ctx[size_t(r)], gx, gy, kx, ky, h, n, n_time, dt, &p));
        else
          check_rc(fpc_problem_create_1d(m->ctx[size_t(r)], gx, kx, h, n, n_time, dt, &p));
        s->prob.push_back(p);
        if (p->generic) throw Unsupported{"sharded solve: power-of-two sizes only"};
        fpc_plan_t pl = nullptr;
        check_rc(fpc_plan_create(p, alpha, &pl));
        s->plan.push_back(pl);
        DeviceGuard g(m->devices[size_t(r)]);
        const size_t c = size_t(s->cs[size_t(r)]), hr = size_t(s->hs[size_t(r)]);
        s->cols.push_back(dalloc<double>(size_t(n_time) * c + 2));
        s->zf.push_back(dalloc<double>(2 * size_t(s->H) * c + 2));
        s->rows.push_back(dalloc<double>(2 * hr * size_t(s->ns) + 2));
        s->zb.push_back(dalloc<double>(2 * size_t(s->H) * c + 2));
        s->zt.push_back(dalloc<double>(size_t(n_time) * c + 2));
      }
    } catch (...) {
      fpc_sharded_destroy(s);
      throw;
    }
    *out = s;
  });
}

int fpc_sharded_create_1d(fpc_multi_t m, double gamma, double kappa, double h, int n_space, int n_time, double dt,
                          double alpha, fpc_sharded_t* out) {
  return sharded_create(m, false, gamma, 0.0, kappa, 0.0, h, n_space, n_time, dt, alpha, out);
}

int fpc_sharded_create_2d(fpc_multi_t m, double gx, double gy, double kx, double ky, double h, int n_per_dim,
                          int n_time, double dt, double alpha, fpc_sharded_t* out) {
  return sharded_create(m, true, gx, gy, kx, ky, h, n_per_dim, n_time, dt, alpha, out);
}

int fpc_sharded_destroy(fpc_sharded_t s) {
  if (!s) return FPC_OK;
  for (size_t r = 0; r < s->prob.size(); ++r) {
    DeviceGuard g(s->m->devices[r]);
    cudaStreamSynchronize(s->m->ctx[r]->stream);
    for (auto* v : {&s->cols, &s->zf, &s->rows, &s->zb, &s->zt})
      if (r < v->size()) cudaFree((*v)[r]);
    if (r < s->plan.size()) fpc_plan_destroy(s->plan[r]);
    fpc_problem_destroy(s->prob[r]);
  }
  delete s;
  return FPC_OK;
}

int fpc_sharded_info(fpc_sharded_t s, int* n_ranks, int* nt_local) {
  if (!s) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  if (n_ranks) *n_ranks = s->G;
  if (nt_local) *nt_local = s->nt_loc;
  return FPC_OK;
}

int fpc_sharded_matvec(fpc_sharded_t s, const double* v, double* out) {
  if (!s || !v || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    SVec a = svec_alloc(s), b = svec_alloc(s);
    try {
      sh_upload(s, v, a);
      sh_matvec(s, a, b);
      sh_download(s, b, out);
    } catch (...) {
      svec_free(s, a);
      svec_free(s, b);
      throw;
    }
    svec_free(s, a);
    svec_free(s, b);
  });
}

int fpc_sharded_pc_apply(fpc_sharded_t s, const double* v, double* out) {
  if (!s || !v || !out) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    SVec a = svec_alloc(s), b = svec_alloc(s);
    try {
      sh_upload(s, v, a);
      sh_pc_apply(s, a, b, 1.0);
      sh_download(s, b, out);
    } catch (...) {
      svec_free(s, a);
      svec_free(s, b);
      throw;
    }
    svec_free(s, a);
    svec_free(s, b);
  });
}

// gmres_right on the sharded operator (krylov.hpp:83-192; the reference's Gram-Schmidt with its
// conditional re-orthogonalisation, as fpc_gmres_callbacks) + GMRES(m) emulation; host b and x.
int fpc_sharded_gmres(fpc_sharded_t s, const double* b, double* x, const fpc_solver_config* cfg_in, fpc_report* report,
                      double* history, int history_cap) {
  if (!s || !b || !x || !cfg_in || !report) return set_err(FPC_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    const fpc_solver_config cfg = *cfg_in;
    if (cfg.max_iter < 0) throw InvalidArg{"gmres_right: max_iter must be non-negative"};
    const int mcyc = (cfg.restart > 0 && cfg.restart < cfg.max_iter) ? cfg.restart : cfg.max_iter;
    if (mcyc + 1 > 250) throw Unsupported{"sharded gmres_right: at most 249 steps per cycle"};
    const auto t0 = std::chrono::steady_clock::now();
    *report = fpc_report{};
    std::vector<SVec> pool;
    auto fresh = [&]() -> SVec* {
      pool.push_back(svec_alloc(s));
      return &pool.back();
    };
    pool.reserve(size_t(mcyc) + 8);
    struct Free {
      fpc_sharded_s* s;
      std::vector<SVec>* p;
      ~Free() {
        for (auto& v : *p) svec_free(s, v);
      }
    } fr{s, &pool};
    SVec* B = fresh();
    SVec* X = fresh();
    SVec* R = fresh();
    SVec* W = fresh();
    SVec* Z = fresh();
    SVec* T = fresh();
    std::vector<SVec*> V;
    for (int i = 0; i <= mcyc; ++i) V.push_back(fresh());
    sh_upload(s, b, *B);
    const double norm_b = std::sqrt(sh_dots(s, {}, *B, true)[0]);
    int total = 0, cycles = 0, reorth = 0, hist_len = 0;
    bool conv = norm_b == 0.0, have_x = false;
    double last_rel = conv ? 0.0 : 1.0, norm_r = norm_b;
    SVec* rhs = B;
    while (!conv && total < cfg.max_iter) {
      const int budget = std::min(mcyc, cfg.max_iter - total);
      const double tol_c = cfg.tol * norm_b / norm_r;
      sh_lincomb(s, {rhs}, {1.0 / norm_r}, *V[0]);
      std::vector<std::vector<double>> Hc;
      std::vector<double> gc, gs, gg{norm_r};
      int steps = 0;
      bool inner = false;
      for (int j = 0; j < budget; ++j) {
        sh_pc_apply(s, *V[size_t(j)], *Z, 1.0);
        sh_matvec(s, *Z, *W);
        std::vector<SVec*> Vj(V.begin(), V.begin() + j + 1);
        std::vector<double> h(size_t(j) + 2, 0.0);
        const double norm_before = std::sqrt(sh_dots(s, {}, *W, true)[0]);
        double norm_w = norm_before;
        for (int pass = 0; pass < 2; ++pass) {  // krylov.hpp:116-131
          const std::vector<double> d = sh_dots(s, Vj, *W, false);
          const double nw2 = sh_update(s, Vj, d, *W);
          for (int i = 0; i <= j; ++i) h[size_t(i)] += d[size_t(i)];
          const double prev = norm_w;
          norm_w = std::sqrt(std::max(nw2, 0.0));
          if (pass == 0 && !(norm_w < 0.70710678118654752 * prev)) break;
          if (pass == 1) ++reorth;
        }
        h[size_t(j) + 1] = norm_w;
        for (int i = 0; i < j; ++i) {
          const double hi = h[size_t(i)], hi1 = h[size_t(i) + 1];
          h[size_t(i)] = gc[size_t(i)] * hi + gs[size_t(i)] * hi1;
          h[size_t(i) + 1] = -gs[size_t(i)] * hi + gc[size_t(i)] * hi1;
        }
        const double rad = std::hypot(h[size_t(j)], h[size_t(j) + 1]);
        const double c_ = rad > 0.0 ? h[size_t(j)] / rad : 1.0, s_ = rad > 0.0 ? h[size_t(j) + 1] / rad : 0.0;
        gc.push_back(c_);
        gs.push_back(s_);
        h[size_t(j)] = rad;
        h[size_t(j) + 1] = 0.0;
        gg.push_back(-s_ * gg[size_t(j)]);
        gg[size_t(j)] *= c_;
        Hc.push_back(h);
        steps = j + 1;
        const double rel_c = std::abs(gg[size_t(j) + 1]) / norm_r;
        last_rel = rel_c * norm_r / norm_b;
        if (history && hist_len < history_cap) history[hist_len] = last_rel;
        ++hist_len;
        if (rel_c <= tol_c) {
          inner = true;
          break;
        }
        if (norm_w <= 1e-14 * std::max(1.0, norm_before)) break;
        sh_lincomb(s, {W}, {1.0 / norm_w}, *V[size_t(j) + 1]);
      }
      total += steps;
      ++cycles;
      if (steps > 0) {
        std::vector<double> y(size_t(steps), 0.0);
        for (int i = steps - 1; i >= 0; --i) {
          double acc = gg[size_t(i)];
          for (int k = i + 1; k < steps; ++k) acc -= Hc[size_t(k)][size_t(i)] * y[size_t(k)];
          y[size_t(i)] = acc / Hc[size_t(i)][size_t(i)];
        }
        std::vector<SVec*> Vs(V.begin(), V.begin() + steps);
        sh_lincomb(s, Vs, y, *W);
        sh_pc_apply(s, *W, *Z, 1.0);  // delta = P^{-1} V y (krylov.hpp:180-183)
        if (have_x) {
          sh_lincomb(s, {X, Z}, {1.0, 1.0}, *T);
          std::swap(X, T);
        } else {
          sh_lincomb(s, {Z}, {1.0}, *X);
          have_x = true;
        }
      }
      if (inner) conv = true;
      if (conv || steps == 0 || total >= cfg.max_iter) break;
      sh_matvec(s, *X, *W);  // r = b - A x
      sh_lincomb(s, {B, W}, {1.0, -1.0}, *R);
      rhs = R;
      norm_r = std::sqrt(sh_dots(s, {}, *R, true)[0]);
      if (norm_r == 0.0) conv = true;
    }
    double trr = 0.0;
    if (!have_x) sh_lincomb(s, {B}, {0.0}, *X);
    if (norm_b > 0.0) {
      sh_matvec(s, *X, *W);
      sh_lincomb(s, {B, W}, {1.0, -1.0}, *R);
      trr = std::sqrt(sh_dots(s, {}, *R, true)[0]) / norm_b;
    }
    sh_download(s, *X, x);
    report->converged = conv ? 1 : 0;
    report->iterations = total;
    report->iterations_exact = double(total);
    report->restarts = cycles > 0 ? cycles - 1 : 0;
    report->reorthogonalizations = reorth;
    report->final_relative_residual = last_rel;
    report->true_relative_residual = trr;
    report->history_len = hist_len;
    report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"
