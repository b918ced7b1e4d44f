// precond.cu — the paper's baseline preconditioners inside the same device-resident PCG loop
// (§3.2): P = I (unpreconditioned CG) and the Jacobi
// preconditioner of Eq 25, (P_Jac)_ii = 1/A_ii.
//
// diag(A) from the octant phases (no assembly): a node's diagonal entry sums the element
// diagonals of its 2^d octants, and every corner of a Q1 element has the same one
//   thermal 3D  K_ref,aa = h/3            thermal 2D  2/3
//   elastic 3D  (K_lam)_aa = h/9, (K_mu)_aa = 4h/9 (every component)
//   elastic 2D  1/3 and 1 (per unit depth)
// (exact 1D integrals: int phi'^2 = 1/h, int phi^2 = h/3).
// One iteration = two fused elementwise passes + K:
//   jac_r: r -= alpha p ; ||r||_inf and gamma_1 = r.(P r) partials          (Alg 2 l.11, l.3, l.5, l.7)
//   jac_d: d = P r + beta d ; u += alpha_prev d_old                          (l.8, l.12)
#include <cuda_runtime.h>

#include "common.cuh"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace uno {

constexpr int JT = 256;

__device__ __forceinline__ unsigned jac_octant_bits(const Ctx& cx, long long i) {
  // periodic or Dirichlet-z node i (stored index): phases of the 2^d voxels around it
  const Geo& g = cx.g;
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const int s1 = __ffs(N1) - 1, s2 = __ffs(N2) - 1;
  const int x = (int)(i & (N1 - 1)), y = (int)((i >> s1) & (N2 - 1));
  const int z = (int)(i >> (s1 + s2)) + g.dirz + g.zlo;
  unsigned bits = 0;
  for (int o = 0; o < (1 << g.dim); ++o) {
    const int ex = (x - 1 + (o & 1)) & (N1 - 1), ey = (y - 1 + ((o >> 1) & 1)) & (N2 - 1);
    const int ez = g.dim == 3 ? ((z - 1 + ((o >> 2) & 1)) & (N3 - 1)) : 0;
    bits |= (__ldg(cx.phase + ((long long)ez * N2 + ey) * N1 + ex) ? 1u : 0u) << o;
  }
  return bits;
}

__global__ void jacobi_dinv_kernel(Ctx cx, double* __restrict__ dinv) {
  const Geo g = cx.g;
  const int no = 1 << g.dim;
  double e0, e1;  // per-octant diagonal contribution of phase 0 / phase 1
  if (g.c == 1) {
    const double w = g.dim == 3 ? g.h / 3.0 : 2.0 / 3.0;
    e0 = w * cx.mat[0][0];
    e1 = w * cx.mat[1][0];
  } else if (g.dim == 3) {
    e0 = g.h / 9.0 * (cx.mat[0][0] + 4.0 * cx.mat[0][1]);
    e1 = g.h / 9.0 * (cx.mat[1][0] + 4.0 * cx.mat[1][1]);
  } else {
    e0 = cx.mat[0][0] / 3.0 + cx.mat[0][1];
    e1 = cx.mat[1][0] / 3.0 + cx.mat[1][1];
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (long long)gridDim.x * blockDim.x) {
    const int n1 = __popc(jac_octant_bits(cx, i));
    dinv[i] = 1.0 / ((no - n1) * e0 + n1 * e1);
  }
}

// r update, ||r||_inf and gamma partials (one CTA partial per slot), or (STANDALONE) z = P r
template <bool JAC, int MODE>
__global__ void __launch_bounds__(JT) jac_r_kernel(Ctx cx, const double* __restrict__ dinv, const double* __restrict__ src,
                                                   double* __restrict__ zout) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE == CG && !st->active) return;
  __shared__ double red_sh[32];
  const long long cn = (long long)g.c * g.n;
  bool upd = false;
  double alpha = 0.0;
  if (MODE == CG) {
    upd = st->iters > 0;
    alpha = st->alpha;
  }
  const double* rin = (MODE == CG ? cx.r : src) + (long long)load * cn;
  double* rr = cx.r + (long long)load * cn;
  const double* pp = cx.p + (long long)load * cn;
  double mx = 0.0, gm = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cn; i += (long long)gridDim.x * blockDim.x) {
    double r = rin[i];
    if (MODE == CG && upd) {
      r = fma(-alpha, pp[i], r);
      rr[i] = r;
    }
    const double z = JAC ? r * dinv[g.c == 1 ? i : i % g.n] : r;
    if (MODE != CG) zout[(long long)load * cn + i] = z;
    mx = fmax(mx, fabs(r));
    gm = fma(r, z, gm);
  }
  if (MODE == CG) partial_write<true>(cx, RED_RNORM, load, blockIdx.x, mx, red_sh);
  __syncthreads();
  partial_write<false>(cx, RED_GAMMA, load, blockIdx.x, gm, red_sh);
}

// KIND 0: s = r (identity), 1: s = r dinv (Jacobi), 2: s read from `aux` (an opaque P r, dirichlet.cu)
template <int KIND>
__global__ void __launch_bounds__(JT) jac_d_kernel(Ctx cx, const double* __restrict__ aux) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  const LoadState* st = cx.st + load;
  if (!st->active) return;
  const long long cn = (long long)g.c * g.n;
  const double* rr = cx.r + (long long)load * cn;
  double* d = cx.d + (long long)load * cn;
  double* u = cx.u + (long long)load * cn;
  const int it0 = st->iters;
  const double beta = st->beta, alpha = st->alpha;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cn; i += (long long)gridDim.x * blockDim.x) {
    const double s = KIND == 2 ? aux[(long long)load * cn + i] : (KIND == 1 ? rr[i] * aux[g.c == 1 ? i : i % g.n] : rr[i]);
    if (it0 == 0) {
      d[i] = s;  // d = s  (Alg 2 l.2, l.8)
    } else {
      const double dold = d[i];
      u[i] = fma(alpha, dold, u[i]);  // deferred u += alpha_{m-1} d_{m-1}  (Alg 2 l.12)
      d[i] = fma(beta, dold, s);
    }
  }
}

static unsigned jac_grid(const Geo& g) {
  const long long cn = (long long)g.c * g.n;
  long long b = (cn + JT - 1) / JT;
  return (unsigned)(b > 148 * 8 ? 148 * 8 : b);
}

int jacobi_nblk(const Geo& g) { return (int)jac_grid(g); }

int launch_jacobi_dinv(const Ctx& cx, double* dinv, cudaStream_t s) {
  long long b = (cx.g.n + 255) / 256;
  jacobi_dinv_kernel<<<(unsigned)(b > 148 * 16 ? 148 * 16 : b), 256, 0, s>>>(cx, dinv);
  return 1;
}

int launch_jac_r(const Ctx& cx, int kind, int mode, const double* dinv, const double* src, double* z, cudaStream_t s) {
  const dim3 grid(jac_grid(cx.g), cx.g.nrhs);
  const bool jac = kind == 2;
  if (mode == CG) {
    if (jac) jac_r_kernel<true, CG><<<grid, JT, 0, s>>>(cx, dinv, src, z);
    else jac_r_kernel<false, CG><<<grid, JT, 0, s>>>(cx, dinv, src, z);
  } else {
    if (jac) jac_r_kernel<true, STANDALONE><<<grid, JT, 0, s>>>(cx, dinv, src, z);
    else jac_r_kernel<false, STANDALONE><<<grid, JT, 0, s>>>(cx, dinv, src, z);
  }
  return 1;
}

int launch_jac_d(const Ctx& cx, int kind, const double* dinv, cudaStream_t s) {
  const dim3 grid(jac_grid(cx.g), cx.g.nrhs);
  if (kind == 2) jac_d_kernel<1><<<grid, JT, 0, s>>>(cx, dinv);
  else jac_d_kernel<0><<<grid, JT, 0, s>>>(cx, dinv);
  return 1;
}

int launch_jac_d_ext(const Ctx& cx, const double* sbuf, cudaStream_t s) {
  const dim3 grid(jac_grid(cx.g), cx.g.nrhs);
  jac_d_kernel<2><<<grid, JT, 0, s>>>(cx, sbuf);
  return 1;
}

}  // namespace uno
