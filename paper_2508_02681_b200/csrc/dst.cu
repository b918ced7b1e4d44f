// dst.cu — DST-I along z for the mixed boundary condition (periodic x, y; Dirichlet z).
//
// PAPER.md Table 1 row "Mixed" uses F^x o T_ST^y in 2D; for 3D with Dirichlet faces on
// z (BASELINE config 4 variant) the unitary transform is U = F_x (x) F_y (x) DST-I_z (SURVEY
// A13; DST variant SPEC S:249).  The z transform is applied FIRST, on the real field, so the
// remaining x/y transforms are the periodic 2D machinery over the N3-1 sine planes.
//
// DST-I of length N-1 (N = N3) through a complex FFT of length 2N of the odd extension
//   y_0 = 0, y_j = x_j (1 <= j < N), y_N = 0, y_{2N-j} = -x_j   =>   sum_j x_j sin(pi j m / N) = (i/2) Y_m.
// Two adjacent real x-columns are packed as one complex column (a double2 of the row), so
// the packed result's real/imaginary parts are the two real transforms.  Unnormalised
// (the sine sum); N/2 of the round trip is folded into the tabulated symbol.
//   dstz_kernel<L2, false, CG>: r -= alpha p ; ||r||_inf ; r_tilde = S_z r        (Alg 2 l.11, l.3, l.4)
//   dstz_kernel<L2, true,  CG>: s = S_z s_tilde ; u += alpha d_old ; d = s + beta d (Alg 2 l.6, 8, 12)
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "dev_common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace uno {

template <int L2>
__host__ __device__ constexpr int dst_smem_bytes() {
  return (8 * L2 + L2) * (int)sizeof(double2);
}

template <int L2, bool INV, int MODE>
__global__ void __launch_bounds__(fft_threads(L2)) dstz_kernel(Ctx cx, const double* __restrict__ src,
                                                               double* __restrict__ dst) {
  constexpr int T = fft_threads(L2);
  constexpr int N = L2 / 2;  // = N3
  constexpr int P3 = N - 1;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  extern __shared__ double2 smem[];
  double2* tile = smem;
  double2* tw = smem + 8 * L2;
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int M = g.N1 / 2;  // double2 per row
  const int nxc = g.N1 / 16;
  const int xc = blockIdx.x % nxc;
  const int yz = blockIdx.x / nxc;
  const int y = yz % g.N2, comp = yz / g.N2;
  const long long rowpitch = (long long)g.N2 * M;  // double2 per z plane
  const long long col0 = ((long long)load * g.c + comp) * P3 * rowpitch + (long long)y * M + xc * 8;
  for (int i = t; i < L2; i += T) tw[i] = cx.tw.z2[i];
  // stage the columns into the odd extension
  double mx = 0.0;
  const double2* s2 = reinterpret_cast<const double2*>(src);
  bool upd = false;
  double alpha = 0.0;
  if (!INV && MODE == CG) {
    upd = st->iters > 0;
    alpha = st->alpha;
  }
  for (int e = t; e < 8 * P3; e += T) {
    const int pz = e >> 3, c = e & 7;
    const long long gi = col0 + (long long)pz * rowpitch + c;
    double2 v = s2[gi];
    if (!INV && MODE == CG && upd) {  // r <- r - alpha p   (Alg 2 l.11)
      const double2 pv = reinterpret_cast<const double2*>(cx.p)[gi];
      v.x = fma(-alpha, pv.x, v.x);
      v.y = fma(-alpha, pv.y, v.y);
      reinterpret_cast<double2*>(cx.r)[gi] = v;
    }
    if (!INV) mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    tile[tidx(pz + 1, c)] = v;
    tile[tidx(L2 - 1 - pz, c)] = make_double2(-v.x, -v.y);
  }
  if (t < 8) {
    tile[tidx(0, t)] = make_double2(0.0, 0.0);
    tile[tidx(N, t)] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_tile<L2, false>(tile, tw);
  // sine coefficients m = 1..N-1: (i/2) Y_m
  if (!INV) {
    double2* o2 = reinterpret_cast<double2*>(dst);
    for (int e = t; e < 8 * P3; e += T) {
      const int pm = e >> 3, c = e & 7;
      const double2 Y = tile[tidx(pm + 1, c)];
      o2[col0 + (long long)pm * rowpitch + c] = make_double2(-0.5 * Y.y, 0.5 * Y.x);
    }
    if (MODE == CG) partial_write<true>(cx, RED_RNORM, load, blockIdx.x, mx, red_sh);
  } else if (MODE != CG) {
    double2* o2 = reinterpret_cast<double2*>(dst);
    for (int e = t; e < 8 * P3; e += T) {
      const int pm = e >> 3, c = e & 7;
      const double2 Y = tile[tidx(pm + 1, c)];
      o2[col0 + (long long)pm * rowpitch + c] = make_double2(-0.5 * Y.y, 0.5 * Y.x);
    }
  } else {
    double2* d2 = reinterpret_cast<double2*>(cx.d);
    double2* u2 = reinterpret_cast<double2*>(cx.u);
    const int it0 = st->iters;
    const double beta = st->beta, alph = st->alpha;
    for (int e = t; e < 8 * P3; e += T) {
      const int pm = e >> 3, c = e & 7;
      const double2 Y = tile[tidx(pm + 1, c)];
      const double2 sv = make_double2(-0.5 * Y.y, 0.5 * Y.x);
      const long long gi = col0 + (long long)pm * rowpitch + c;
      if (it0 == 0) {
        d2[gi] = sv;
      } else {
        const double2 dold = d2[gi];
        double2 uu = u2[gi];
        uu.x = fma(alph, dold.x, uu.x);
        uu.y = fma(alph, dold.y, uu.y);
        u2[gi] = uu;
        d2[gi] = make_double2(fma(beta, dold.x, sv.x), fma(beta, dold.y, sv.y));
      }
    }
  }
}

// ---------------------------------------------------------------------- slab pencils, Dirichlet z
// In slab mode the z transform runs on the complex pencil [lc][kx][z][yc] (after the x/y FFTs and
// the all-to-all; the transforms commute, U is the same).  Storage is padded: node plane 0 is the
// fixed Dirichlet face (always 0) and sine mode m = 1..N3-1 is kept at index m, index 0 = 0.  The
// DST-I of a complex column is the same odd-extension FFT: (i/2) Y_m gives S(a) + i S(b).
template <int L2>
__global__ void __launch_bounds__(fft_threads(L2)) pencil_dst_kernel(Ctx cx, double2* __restrict__ P) {
  constexpr int T = fft_threads(L2);
  constexpr int N = L2 / 2;  // = N3
  const Geo g = cx.g;        // pencil view: N2 := Yc, N3 global
  const int load = blockIdx.y;
  if (!cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tile = smem;
  double2* tw = smem + 8 * L2;
  const int t = threadIdx.x;
  const int Yc = g.N2, nyc = Yc / 8;
  const int yq = blockIdx.x % nyc;
  const long long lk = blockIdx.x / nyc;  // (component, kx) row of this load
  const long long col0 = ((long long)load * g.c * g.H1 + lk) * N * Yc + yq * 8;
  for (int i = t; i < L2; i += T) tw[i] = cx.tw.z2[i];
  for (int e = t; e < 8 * (N - 1); e += T) {
    const int pz = (e >> 3) + 1, c = e & 7;
    const double2 v = P[col0 + (long long)pz * Yc + c];
    tile[tidx(pz, c)] = v;
    tile[tidx(L2 - pz, c)] = make_double2(-v.x, -v.y);
  }
  if (t < 8) {
    tile[tidx(0, t)] = make_double2(0.0, 0.0);
    tile[tidx(N, t)] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_tile<L2, false>(tile, tw);
  for (int e = t; e < 8 * N; e += T) {
    const int m = e >> 3, c = e & 7;
    const double2 Y = tile[tidx(m, c)];
    P[col0 + (long long)m * Yc + c] = m == 0 ? make_double2(0.0, 0.0) : make_double2(-0.5 * Y.y, 0.5 * Y.x);
  }
}

// s_hat = G_hat r_hat on every bin of the pencil (all c components of a bin together) and the
// Parseval partial of gamma (weights of the R2C kx planes), grid-stride over the bins.
constexpr int PG_NBLK = 148 * 4;
template <int NC>
__global__ void __launch_bounds__(256) pencil_gmul_kernel(Ctx cx, double2* __restrict__ P) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (!cx.st[load].active) return;
  __shared__ double red_sh[32];
  const long long ns = g.nspec, zy = (long long)g.N3 * g.N2;
  double2* base = P + (long long)load * g.c * ns;
  double part = 0.0;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < ns; b += (long long)gridDim.x * blockDim.x) {
    double2 x[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) x[q] = base[q * ns + b];
    part += gmul_vals<NC>(x, cx.gtab, ns, b, parseval_w((int)(b / zy), g.M));
#pragma unroll
    for (int q = 0; q < NC; ++q) base[q * ns + b] = x[q];
  }
  partial_write<false>(cx, RED_GAMMA, load, blockIdx.x, part, red_sh);
}

int pencil_gmul_nblk() { return PG_NBLK; }

template <class F>
static int dispatch_l2(int L, F&& f);

// z . G . z^-1 of a Dirichlet-z slab pencil (in place): DST-I, symbol multiply + gamma partial, DST-I.
int launch_pencil_dst_green(const Ctx& cx, double2* pencil, cudaStream_t s) {
  const Geo& g = cx.g;
  if (!g.zpad || g.N2 % 8) return -1;
  const int r = dispatch_l2(2 * g.N3, [&](auto Lc) {
    constexpr int L2 = decltype(Lc)::value;
    const dim3 grid((unsigned)((long long)g.c * g.H1 * (g.N2 / 8)), g.nrhs);
    const int sm = dst_smem_bytes<L2>();
    if (sm > 48 * 1024) cudaFuncSetAttribute(pencil_dst_kernel<L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    pencil_dst_kernel<L2><<<grid, fft_threads(L2), sm, s>>>(cx, pencil);
    const dim3 gg(PG_NBLK, g.nrhs);
    if (g.c == 1) pencil_gmul_kernel<1><<<gg, 256, 0, s>>>(cx, pencil);
    else pencil_gmul_kernel<3><<<gg, 256, 0, s>>>(cx, pencil);
    pencil_dst_kernel<L2><<<grid, fft_threads(L2), sm, s>>>(cx, pencil);
    return 3;
  });
  return r;
}

template <class F>
static int dispatch_l2(int L, F&& f) {
  switch (L) {
    case 16: return f(std::integral_constant<int, 16>{});
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 128: return f(std::integral_constant<int, 128>{});
    case 256: return f(std::integral_constant<int, 256>{});
    case 512: return f(std::integral_constant<int, 512>{});
    case 1024: return f(std::integral_constant<int, 1024>{});
    default: return -1;
  }
}

int launch_dstz(const Ctx& cx, int mode, bool inverse, const double* src, double* dst, cudaStream_t s) {
  const Geo& g = cx.g;
  if (!g.dirz || g.N1 < 16) return -1;
  return dispatch_l2(2 * g.N3, [&](auto Lc) {
    constexpr int L2 = decltype(Lc)::value;
    const dim3 grid((unsigned)(g.c * g.N2 * (g.N1 / 16)), g.nrhs);
    const int sm = dst_smem_bytes<L2>();
    auto go = [&](auto k) {
      if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      k<<<grid, fft_threads(L2), sm, s>>>(cx, src, dst);
      return 1;
    };
    if (!inverse) return mode == CG ? go(dstz_kernel<L2, false, CG>) : go(dstz_kernel<L2, false, STANDALONE>);
    return mode == CG ? go(dstz_kernel<L2, true, CG>) : go(dstz_kernel<L2, true, STANDALONE>);
  });
}

}  // namespace uno
