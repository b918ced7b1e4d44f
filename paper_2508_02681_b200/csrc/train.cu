// train.cu — second-order UNO preconditioner training on the GPU (§4.4 Alg 4, Eq 62-72,
// App. B.1-B.2).  3D periodic grids, T = DFT, c = 1 or 3.
//
// Features (Eq 62, 67, B.2): every training pair (r, s) is transformed once with the library's
// own forward passes (x R2C, y FFT, z FFT; unnormalised, so products carry 1/n), and per half-
// spectrum bin the C alpha's and C beta's are accumulated (Eq B7 order of the unique entries).
// Newton (Alg 4): v(k) = psi(theta_0) + [k in K] psi(theta_p(k)), K = {|k_i| <= M}, conjugate
// pairs {k, -k} share theta_p; loss L = sum_k w_k (1/2 v^T H(alpha) v - beta . v) + delta with the
// Parseval weights w_k of the half spectrum (1 on the k_x = 0, N1/2 planes, else 2).  One epoch:
//   train_bin_kernel    all bins: g_0, H_00 (J_0^T H J_0 + gv . D2) and loss partials
//   train_pair_kernel   pairs: g_p, H_pp, H_0p; H_pp^-1; Schur partials H_0p H_pp^-1 H_0p^T, H_0p H_pp^-1 g_p
//   train_solve_kernel  1 thread: fixed-order sums, S d_0 = g_0 - sum(...) (Gauss-Jordan), loss
//   train_update_kernel pairs: d_p = H_pp^-1 (g_p - H_0p^T d_0), theta_p <- theta_p - t d_p
// with the step halved while the loss increases (reading R15, as the oracle).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/uno_cg.h"
#include "common.cuh"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace uno {

// ---- local parametrization psi (Eq 45 c=1 form t^2, Eq B5 c=3) and its derivatives -------------
template <int C>
__device__ __forceinline__ void psi_v(const double* t, double* v) {
  if (C == 1) {
    v[0] = t[0] * t[0];
  } else {
    v[0] = t[0] * t[0];
    v[1] = t[1] * t[1] + t[2] * t[2];
    v[2] = t[0] * t[2];
    v[3] = t[3] * t[3] + t[4] * t[4] + t[5] * t[5];
    v[4] = t[1] * t[4] + t[2] * t[5];
    v[5] = t[0] * t[5];
  }
}
// J[m][i] = d v_m / d t_i
template <int C>
__device__ __forceinline__ void psi_J(const double* t, double J[C][C]) {
  for (int m = 0; m < C; ++m)
    for (int i = 0; i < C; ++i) J[m][i] = 0.0;
  if (C == 1) {
    J[0][0] = 2 * t[0];
  } else {
    J[0][0] = 2 * t[0];
    J[1][1] = 2 * t[1];
    J[1][2] = 2 * t[2];
    J[2][0] = t[2];
    J[2][2] = t[0];
    J[3][3] = 2 * t[3];
    J[3][4] = 2 * t[4];
    J[3][5] = 2 * t[5];
    J[4][1] = t[4];
    J[4][2] = t[5];
    J[4][4] = t[1];
    J[4][5] = t[2];
    J[5][0] = t[5];
    J[5][5] = t[0];
  }
}
// sum_m g_m d2 v_m / dt_i dt_k (psi is quadratic: constant second derivatives)
template <int C>
__device__ __forceinline__ void psi_D2g(const double* g, double D[C][C]) {
  for (int i = 0; i < C; ++i)
    for (int k = 0; k < C; ++k) D[i][k] = 0.0;
  if (C == 1) {
    D[0][0] = 2 * g[0];
  } else {
    D[0][0] += 2 * g[0];
    D[1][1] += 2 * g[1];
    D[2][2] += 2 * g[1];
    D[0][2] += g[2];
    D[2][0] += g[2];
    D[3][3] += 2 * g[3];
    D[4][4] += 2 * g[3];
    D[5][5] += 2 * g[3];
    D[1][4] += g[4];
    D[4][1] += g[4];
    D[2][5] += g[4];
    D[5][2] += g[4];
    D[0][5] += g[5];
    D[5][0] += g[5];
  }
}
// H(alpha) = d^2 l / dv dv (Eq 66, App. B.2), alpha in Eq B7 order
template <int C>
__device__ __forceinline__ void hess_alpha(const double* a, double H[C][C]) {
  if (C == 1) {
    H[0][0] = 2 * a[0];
  } else {
    const double a1 = a[0], a2 = a[1], a3 = a[2], a4 = a[3], a5 = a[4], a6 = a[5];
    const double R[6][6] = {{2 * a1, 0, a3, 0, 0, a6},
                            {0, 2 * a2, a3, 0, a5, 0},
                            {a3, a3, 2 * (a1 + a2), 0, a6, a5},
                            {0, 0, 0, 2 * a4, a5, a6},
                            {0, a5, a6, a5, 2 * (a2 + a4), a3},
                            {a6, 0, a5, a6, a3, 2 * (a1 + a4)}};
    for (int m = 0; m < C; ++m)
      for (int n = 0; n < C; ++n) H[m][n] = R[m][n];
  }
}
// in-place inverse of a small SPD-ish matrix (Gauss-Jordan with partial pivoting)
template <int C>
__device__ __forceinline__ void inv_small(double A[C][C], double X[C][C]) {
  for (int i = 0; i < C; ++i)
    for (int j = 0; j < C; ++j) X[i][j] = i == j ? 1.0 : 0.0;
  for (int col = 0; col < C; ++col) {
    int piv = col;
    for (int r = col + 1; r < C; ++r)
      if (fabs(A[r][col]) > fabs(A[piv][col])) piv = r;
    if (piv != col)
      for (int j = 0; j < C; ++j) {
        double t = A[col][j];
        A[col][j] = A[piv][j];
        A[piv][j] = t;
        t = X[col][j];
        X[col][j] = X[piv][j];
        X[piv][j] = t;
      }
    const double d = 1.0 / A[col][col];
    for (int j = 0; j < C; ++j) {
      A[col][j] *= d;
      X[col][j] *= d;
    }
    for (int r = 0; r < C; ++r)
      if (r != col) {
        const double f = A[r][col];
        for (int j = 0; j < C; ++j) {
          A[r][j] -= f * A[col][j];
          X[r][j] -= f * X[col][j];
        }
      }
  }
}

// per bin: v, gv = H v - beta, H  (feat: [2C][nspec], alpha then beta)
template <int C>
__device__ __forceinline__ void bin_terms(const double* feat, long long ns, long long b, const double* v, double* gv,
                                          double H[C][C]) {
  double a[C], be[C];
  for (int m = 0; m < C; ++m) {
    a[m] = feat[m * ns + b];
    be[m] = feat[(C + m) * ns + b];
  }
  hess_alpha<C>(a, H);
  for (int m = 0; m < C; ++m) {
    double acc = -be[m];
    for (int n = 0; n < C; ++n) acc += H[m][n] * v[n];
    gv[m] = acc;
  }
}

// ---- features ---------------------------------------------------------------------------------
template <int C>
__global__ void train_feat_kernel(Ctx cx, const double2* __restrict__ sr, const double2* __restrict__ ss, double scale,
                                  double* __restrict__ feat) {
  const Geo g = cx.g;
  const long long ns = g.nspec;
  const int c = C == 1 ? 1 : 3;
  const int pa[6] = {0, 1, 0, 2, 1, 0}, pb[6] = {0, 1, 1, 2, 2, 2};  // Eq B7 order
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < ns; b += (long long)gridDim.x * blockDim.x) {
    double al[C], be[C];
    for (int m = 0; m < C; ++m) al[m] = be[m] = 0.0;
    for (int l = 0; l < g.nrhs; ++l) {
      double2 r[3], s[3];
      for (int q = 0; q < c; ++q) {
        r[q] = sr[((long long)l * c + q) * ns + b];
        s[q] = ss[((long long)l * c + q) * ns + b];
      }
      for (int m = 0; m < C; ++m) {
        const int a_ = pa[m], b_ = pb[m];
        const double raRb = r[a_].x * r[b_].x + r[a_].y * r[b_].y;  // Re(conj r_a r_b)
        const double raSb = r[a_].x * s[b_].x + r[a_].y * s[b_].y;
        const double rbSa = r[b_].x * s[a_].x + r[b_].y * s[a_].y;
        al[m] += a_ == b_ ? raRb : 2.0 * raRb;   // alpha_m (Eq 67, B.2)
        be[m] += a_ == b_ ? 2.0 * raSb : 2.0 * (raSb + rbSa);
      }
    }
    for (int m = 0; m < C; ++m) {
      feat[m * ns + b] += scale * al[m];
      feat[(C + m) * ns + b] += scale * be[m];
    }
  }
}

// ---- one Newton epoch ---------------------------------------------------------------------------
struct TrainDev {
  const double* feat;  // [2C][nspec]
  const int* pbin;     // [npair][2] half-spectrum bins of each pair (second -1 if none)
  const int* binpair;  // [nspec] pair of a bin or -1
  const double* th0;   // [C] theta_0
  const double* ths;   // [npair][C]
  double* pst;         // per pair: [C] Hinv g_p, [C][C] Hinv H_0p^T
  double* part;        // partials: [nblk][C + C*C + 1] (bins) then [nblk][C + C*C] (pairs)
  int npair;
};

template <int C>
__device__ __forceinline__ void vbin(const TrainDev& T, long long b, double* v) {
  double t0[C];
  for (int m = 0; m < C; ++m) t0[m] = T.th0[m];
  psi_v<C>(t0, v);
  const int p = T.binpair[b];
  if (p >= 0) {
    double vp[C];
    psi_v<C>(T.ths + (long long)p * C, vp);
    for (int m = 0; m < C; ++m) v[m] += vp[m];
  }
}

template <int C, bool LOSS_ONLY>
__global__ void __launch_bounds__(256) train_bin_kernel(Ctx cx, TrainDev T) {
  const Geo g = cx.g;
  const long long ns = g.nspec;
  constexpr int NP = C + C * C + 1;
  __shared__ double sh[32];
  double J0[C][C];
  psi_J<C>(T.th0, J0);
  double acc[NP];
  for (int i = 0; i < NP; ++i) acc[i] = 0.0;
  const int s2 = __ffs(g.N2) - 1, s3 = __ffs(g.N3) - 1;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < ns; b += (long long)gridDim.x * blockDim.x) {
    const int kx = (int)(b >> (s2 + s3));
    const double w = parseval_w(kx, g.M);
    double v[C], gv[C], H[C][C];
    vbin<C>(T, b, v);
    bin_terms<C>(T.feat, ns, b, v, gv, H);
    // loss: 1/2 v^T H v - beta.v = 1/2 (v . (gv + beta)) - beta . v = 1/2 v.gv - 1/2 beta.v
    double l = 0.0;
    for (int m = 0; m < C; ++m) l += 0.5 * v[m] * (gv[m] - T.feat[(C + m) * ns + b]);
    acc[NP - 1] += w * l;
    if (!LOSS_ONLY) {
      double D[C][C];
      psi_D2g<C>(gv, D);
      for (int i = 0; i < C; ++i) {
        double gi = 0.0;
        for (int m = 0; m < C; ++m) gi += J0[m][i] * gv[m];
        acc[i] += w * gi;
        for (int k = 0; k < C; ++k) {
          double h = D[i][k];
          for (int m = 0; m < C; ++m) {
            double hj = 0.0;
            for (int n = 0; n < C; ++n) hj += H[m][n] * J0[n][k];
            h += J0[m][i] * hj;
          }
          acc[C + i * C + k] += w * h;
        }
      }
    }
  }
  for (int i = 0; i < NP; ++i) {
    if (LOSS_ONLY && i < NP - 1) continue;
    const double bsum = block_reduce<false>(acc[i], sh);
    if (threadIdx.x == 0) T.part[(long long)blockIdx.x * NP + i] = bsum;
    __syncthreads();
  }
}

template <int C>
__global__ void __launch_bounds__(128) train_pair_kernel(Ctx cx, TrainDev T, double* ppart) {
  const Geo g = cx.g;
  const long long ns = g.nspec;
  constexpr int NQ = C + C * C;
  __shared__ double sh[32];
  double J0[C][C];
  psi_J<C>(T.th0, J0);
  double acc[NQ];
  for (int i = 0; i < NQ; ++i) acc[i] = 0.0;
  const int s2 = __ffs(g.N2) - 1, s3 = __ffs(g.N3) - 1;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < T.npair; p += gridDim.x * blockDim.x) {
    double Jp[C][C];
    psi_J<C>(T.ths + (long long)p * C, Jp);
    double gp[C], Hpp[C][C], H0p[C][C];
    for (int i = 0; i < C; ++i) {
      gp[i] = 0.0;
      for (int k = 0; k < C; ++k) Hpp[i][k] = H0p[i][k] = 0.0;
    }
    for (int q = 0; q < 2; ++q) {
      const int bq = T.pbin[2 * p + q];
      if (bq < 0) continue;
      const long long b = bq;
      const double w = parseval_w((int)(b >> (s2 + s3)), g.M);
      double v[C], gv[C], H[C][C], D[C][C];
      vbin<C>(T, b, v);
      bin_terms<C>(T.feat, ns, b, v, gv, H);
      psi_D2g<C>(gv, D);
      for (int i = 0; i < C; ++i) {
        double gi = 0.0;
        for (int m = 0; m < C; ++m) gi += Jp[m][i] * gv[m];
        gp[i] += w * gi;
        for (int k = 0; k < C; ++k) {
          double hpp = D[i][k], h0p = 0.0;
          for (int m = 0; m < C; ++m) {
            double hj = 0.0;
            for (int n = 0; n < C; ++n) hj += H[m][n] * Jp[n][k];
            hpp += Jp[m][i] * hj;
            h0p += J0[m][i] * hj;
          }
          Hpp[i][k] += w * hpp;
          H0p[i][k] += w * h0p;
        }
      }
    }
    double Hi[C][C];
    inv_small<C>(Hpp, Hi);
    // per pair: Hinv g_p and Hinv H_0p^T ; Schur partials
    double* ps = T.pst + (long long)p * NQ;
    for (int i = 0; i < C; ++i) {
      double x = 0.0;
      for (int k = 0; k < C; ++k) x += Hi[i][k] * gp[k];
      ps[i] = x;
      for (int j = 0; j < C; ++j) {  // (Hinv H0p^T)[i][j] = sum_k Hi[i][k] H0p[j][k]
        double y = 0.0;
        for (int k = 0; k < C; ++k) y += Hi[i][k] * H0p[j][k];
        ps[C + i * C + j] = y;
      }
    }
    for (int i = 0; i < C; ++i) {
      double r = 0.0;
      for (int k = 0; k < C; ++k) r += H0p[i][k] * ps[k];  // H0p Hinv g_p
      acc[i] += r;
      for (int l = 0; l < C; ++l) {
        double s = 0.0;
        for (int k = 0; k < C; ++k) s += H0p[i][k] * ps[C + k * C + l];  // H0p Hinv H0p^T
        acc[C + i * C + l] += s;
      }
    }
  }
  for (int i = 0; i < NQ; ++i) {
    const double bsum = block_reduce<false>(acc[i], sh);
    if (threadIdx.x == 0) ppart[(long long)blockIdx.x * NQ + i] = bsum;
    __syncthreads();
  }
}

// fixed-order reductions + the C x C Schur solve; out: [C] d0, [1] loss (without delta)
template <int C>
__global__ void train_solve_kernel(const double* bpart, int nb, const double* ppart, int np, int loss_only, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  constexpr int NP = C + C * C + 1, NQ = C + C * C;
  double tot[NP], sch[NQ];
  for (int i = 0; i < NP; ++i) tot[i] = 0.0;
  for (int i = 0; i < NQ; ++i) sch[i] = 0.0;
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < NP; ++i) tot[i] += bpart[(long long)b * NP + i];
  out[C] = tot[NP - 1];
  if (loss_only) return;
  for (int b = 0; b < np; ++b)
    for (int i = 0; i < NQ; ++i) sch[i] += ppart[(long long)b * NQ + i];
  double S[C][C], Si[C][C], r[C];
  for (int i = 0; i < C; ++i) {
    r[i] = tot[i] - sch[i];
    for (int k = 0; k < C; ++k) S[i][k] = tot[C + i * C + k] - sch[C + i * C + k];
  }
  inv_small<C>(S, Si);
  for (int i = 0; i < C; ++i) {
    double d = 0.0;
    for (int k = 0; k < C; ++k) d += Si[i][k] * r[k];
    out[i] = d;
  }
}

// candidate: theta_0' = theta_0 - t d0 ; theta_p' = theta_p - t (Hinv g_p - Hinv H0p^T d0)
template <int C>
__global__ void train_update_kernel(const double* pst, const double* th0, const double* ths, const double* d0, double t,
                                    int npair, double* th0c, double* thsc) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0)
    for (int i = 0; i < C; ++i) th0c[i] = th0[i] - t * d0[i];
  if (p >= npair) return;
  const double* ps = pst + (long long)p * (C + C * C);
  for (int i = 0; i < C; ++i) {
    double dp = ps[i];
    for (int j = 0; j < C; ++j) dp -= ps[C + i * C + j] * d0[j];
    thsc[(long long)p * C + i] = ths[(long long)p * C + i] - t * dp;
  }
}

// install: gtab[m][b] = v_m(b) / n, G(0) = 0 (shares the periodic null space)
template <int C>
__global__ void train_install_kernel(Ctx cx, TrainDev T, double* gtab) {
  const Geo g = cx.g;
  const long long ns = g.nspec;
  const double inv_n = 1.0 / (double)g.n;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < ns; b += (long long)gridDim.x * blockDim.x) {
    double v[C];
    vbin<C>(T, b, v);
    for (int m = 0; m < C; ++m) gtab[m * ns + b] = b == 0 ? 0.0 : v[m] * inv_n;
  }
}

// ---- launchers ----------------------------------------------------------------------------------
int launch_train_feat(const Ctx& cx, const double2* sr, const double2* ss, double scale, double* feat, cudaStream_t s) {
  const long long ns = cx.g.nspec;
  long long nb = (ns + 255) / 256;
  nb = nb > 148 * 8 ? 148 * 8 : nb;
  if (cx.g.c == 1) train_feat_kernel<1><<<(unsigned)nb, 256, 0, s>>>(cx, sr, ss, scale, feat);
  else train_feat_kernel<6><<<(unsigned)nb, 256, 0, s>>>(cx, sr, ss, scale, feat);
  return 1;
}

}  // namespace uno

namespace uno {

// K = {|k_i| <= M} on the full grid; pairs {k, -k} ordered by canon(k) = min(flat(k), flat(-k))
// (flat = (kz N2 + ky) N1 + kx, as oracle/training.mode_pairs); each pair lists its half-spectrum
// bins (layout [kx][kz][ky]): one for 0 < kx < N1/2, else k and -k (one if self-conjugate).
void train_build_pairs(const Geo& g, int M, std::vector<int>& pbin, std::vector<int>& binpair) {
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3, H = N1 / 2;
  auto sgn = [](int k, int N) { return 2 * k < N ? k : k - N; };  // fftfreq convention: -N/2 is negative
  auto flat = [&](int kx, int ky, int kz) { return ((long long)kz * N2 + ky) * N1 + kx; };
  std::vector<std::pair<long long, int>> reps;  // (canon, unused)
  for (int kz = 0; kz < N3; ++kz)
    for (int ky = 0; ky < N2; ++ky)
      for (int kx = 0; kx < N1; ++kx) {
        if (std::abs(sgn(kx, N1)) > M || std::abs(sgn(ky, N2)) > M || std::abs(sgn(kz, N3)) > M) continue;
        const long long f = flat(kx, ky, kz), fm = flat((N1 - kx) % N1, (N2 - ky) % N2, (N3 - kz) % N3);
        if (f <= fm) reps.push_back({f, 0});
      }
  std::sort(reps.begin(), reps.end());
  pbin.assign(2 * reps.size(), -1);
  binpair.assign((size_t)g.nspec, -1);
  for (size_t p = 0; p < reps.size(); ++p) {
    const long long f = reps[p].first;
    const int kx = (int)(f % N1), ky = (int)((f / N1) % N2), kz = (int)(f / ((long long)N1 * N2));
    const int mx = (N1 - kx) % N1, my = (N2 - ky) % N2, mz = (N3 - kz) % N3;
    int q = 0;
    auto add = [&](int x, int y, int z) {
      if (x > H) return;
      const int b = (int)(((long long)x * N3 + z) * N2 + y);
      if (q == 1 && pbin[2 * p] == b) return;  // self-conjugate
      pbin[2 * p + q++] = b;
      binpair[b] = (int)p;
    };
    add(kx, ky, kz);
    add(mx, my, mz);
  }
}

// Alg 4 on the device: `epochs` Newton steps with backtracking; th0 (host, C), d_ths [npair][C].
int train_newton_run(const Ctx& cx, const double* feat, const std::vector<int>& pbin, const std::vector<int>& binpair,
                     int epochs, double* th0_host, double* d_ths, double* loss_hist, cudaStream_t s, std::string& err) {
  const Geo& g = cx.g;
  const int C = g.c == 1 ? 1 : 6;
  const int npair = (int)(pbin.size() / 2);
  const int NP = C + C * C + 1, NQ = C + C * C;
  const int nb = 148 * 4, npb = npair > 0 ? std::min(148 * 4, (npair + 127) / 128) : 1;
  int *d_pbin = nullptr, *d_binpair = nullptr;
  double *d_th0 = nullptr, *d_th0c = nullptr, *d_thsc = nullptr, *d_pst = nullptr, *d_bpart = nullptr,
         *d_ppart = nullptr, *d_out = nullptr;
  auto al = [&](void** p, size_t bytes) { return cudaMallocAsync(p, bytes ? bytes : 8, s); };
  cudaError_t e;
  if ((e = al((void**)&d_pbin, pbin.size() * 4)) || (e = al((void**)&d_binpair, binpair.size() * 4)) ||
      (e = al((void**)&d_th0, C * 8)) || (e = al((void**)&d_th0c, C * 8)) ||
      (e = al((void**)&d_thsc, (size_t)npair * C * 8)) || (e = al((void**)&d_pst, (size_t)npair * NQ * 8)) ||
      (e = al((void**)&d_bpart, (size_t)nb * NP * 8)) || (e = al((void**)&d_ppart, (size_t)npb * NQ * 8)) ||
      (e = al((void**)&d_out, (C + 1) * 8))) {
    err = cudaGetErrorString(e);
    return -1;
  }
  cudaMemcpyAsync(d_pbin, pbin.data(), pbin.size() * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_binpair, binpair.data(), binpair.size() * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_th0, th0_host, C * 8, cudaMemcpyHostToDevice, s);
  TrainDev T{feat, d_pbin, d_binpair, d_th0, d_ths, d_pst, d_bpart, npair};
  double out[7];
  auto loss_at = [&](const TrainDev& TT) -> double {  // loss (without delta) of the weights in TT
    if (C == 1) train_bin_kernel<1, true><<<nb, 256, 0, s>>>(cx, TT);
    else train_bin_kernel<6, true><<<nb, 256, 0, s>>>(cx, TT);
    if (C == 1) train_solve_kernel<1><<<1, 1, 0, s>>>(d_bpart, nb, d_ppart, npb, 1, d_out);
    else train_solve_kernel<6><<<1, 1, 0, s>>>(d_bpart, nb, d_ppart, npb, 1, d_out);
    cudaMemcpyAsync(out, d_out, (C + 1) * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return out[C];
  };
  double cur = loss_at(T);
  if (loss_hist) loss_hist[0] = cur;
  for (int ep = 0; ep < epochs; ++ep) {
    // gradient / Hessian assembly and the Schur solve for d0 (Alg 4 l.4-6)
    if (C == 1) {
      train_bin_kernel<1, false><<<nb, 256, 0, s>>>(cx, T);
      if (npair) train_pair_kernel<1><<<npb, 128, 0, s>>>(cx, T, d_ppart);
      else cudaMemsetAsync(d_ppart, 0, NQ * 8, s);
      train_solve_kernel<1><<<1, 1, 0, s>>>(d_bpart, nb, d_ppart, npb, 0, d_out);
    } else {
      train_bin_kernel<6, false><<<nb, 256, 0, s>>>(cx, T);
      if (npair) train_pair_kernel<6><<<npb, 128, 0, s>>>(cx, T, d_ppart);
      else cudaMemsetAsync(d_ppart, 0, NQ * 8, s);
      train_solve_kernel<6><<<1, 1, 0, s>>>(d_bpart, nb, d_ppart, npb, 0, d_out);
    }
    // backtracking on the step length (reading R15): theta <- theta - t (d0, dp)
    double t = 1.0;
    TrainDev Tc = T;
    Tc.th0 = d_th0c;
    Tc.ths = d_thsc;
    for (int k = 0; k < 30; ++k) {
      const unsigned ub = (unsigned)std::max(1, (npair + 255) / 256);
      if (C == 1) train_update_kernel<1><<<ub, 256, 0, s>>>(d_pst, d_th0, d_ths, d_out, t, npair, d_th0c, d_thsc);
      else train_update_kernel<6><<<ub, 256, 0, s>>>(d_pst, d_th0, d_ths, d_out, t, npair, d_th0c, d_thsc);
      const double cand = loss_at(Tc);
      if (cand <= cur) {  // accept (no decrease after 30 halvings: stationary to round-off, keep theta)
        cudaMemcpyAsync(d_th0, d_th0c, C * 8, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(d_ths, d_thsc, (size_t)npair * C * 8, cudaMemcpyDeviceToDevice, s);
        cur = cand;
        break;
      }
      t *= 0.5;
    }
    if (loss_hist) loss_hist[ep + 1] = cur;
  }
  cudaMemcpyAsync(th0_host, d_th0, C * 8, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  void* bufs[] = {d_pbin, d_binpair, d_th0, d_th0c, d_thsc, d_pst, d_bpart, d_ppart, d_out};
  for (void* b : bufs) cudaFreeAsync(b, s);
  if (e != cudaSuccess) {
    err = cudaGetErrorString(e);
    return -1;
  }
  return 0;
}

int train_install_run(const Ctx& cx, const std::vector<int>& pbin, const std::vector<int>& binpair,
                      const double* th0_host, const double* d_ths, double* gtab, cudaStream_t s) {
  const Geo& g = cx.g;
  const int C = g.c == 1 ? 1 : 6;
  int* d_binpair = nullptr;
  double* d_th0 = nullptr;
  if (cudaMallocAsync((void**)&d_binpair, binpair.size() * 4, s) != cudaSuccess ||
      cudaMallocAsync((void**)&d_th0, C * 8, s) != cudaSuccess)
    return -1;
  cudaMemcpyAsync(d_binpair, binpair.data(), binpair.size() * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_th0, th0_host, C * 8, cudaMemcpyHostToDevice, s);
  TrainDev T{nullptr, nullptr, d_binpair, d_th0, d_ths, nullptr, nullptr, (int)(pbin.size() / 2)};
  long long nb = (g.nspec + 255) / 256;
  nb = nb > 148 * 8 ? 148 * 8 : nb;
  if (C == 1) train_install_kernel<1><<<(unsigned)nb, 256, 0, s>>>(cx, T, gtab);
  else train_install_kernel<6><<<(unsigned)nb, 256, 0, s>>>(cx, T, gtab);
  cudaFreeAsync(d_binpair, s);
  cudaFreeAsync(d_th0, s);
  return 1;
}

}  // namespace uno
