// kernels.cu — the UNO-CG hot path on B200 (sm_100a), fp64.
//
// Per PCG iteration (Alg 2) five transform passes and one stencil
// kernel run, with the CG vector updates fused into them:
//   F1 xfwd  (CG):  r -= alpha p ; ||r||_inf ; x-axis R2C FFT           (Alg 2 l.11, l.3, l.4)
//   F2 ypass (fwd): y-axis complex FFT                                   (l.4)
//   F3 gpass:       z FFT -> s_hat = G_hat r_hat, gamma_1 (Parseval) -> inverse z FFT
//                                                                        (l.4-7, Eq 46/49)
//   F4 ypass (inv): y-axis inverse FFT                                   (l.6)
//   F5 xinv  (CG):  x-axis C2R -> s ; u += alpha_prev d_old ; d = s + beta d   (l.6, 8, 12)
//   K  kapply (CG): p = A d (matrix-free Q1 gather, no atomics) ; d.p ; alpha  (l.9-10)
// Scalars (alpha, beta, gamma, ||r||) are produced on the device by the last CTA of the
// reducing kernel (deterministic fixed-order combine), so the host never waits inside the
// loop.  In 2D the G pass runs along y directly after F1 (3 passes).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"
#include "dev_common.cuh"

// minimum resident CTAs per SM requested from ptxas for the 256-point passes (occupancy experiments)
// first-stage twiddles of the register-direct y passes read through L1 instead of a per-CTA smem copy:
// faster for the 512-point pass (8 KB table per 4-row CTA: 1204 vs 1238 us at 512^3 elastic), slower for
// the 256-point pass (147 vs 127 us at 256^3 x 3 loads: 15 more LDG per thread in the LSU pipe of a pass
// that runs at 6.3 TB/s)
#ifndef UNO_SERP
#define UNO_SERP 1  // L2-aware launch order of the y / G passes (0: A/B)
#endif
#ifndef UNO_TWLDG_256
#define UNO_TWLDG_256 0
#endif
#ifndef UNO_TWLDG_512
#define UNO_TWLDG_512 1
#endif
#ifndef UNO_YMINB
#define UNO_YMINB 1
#endif
#ifndef UNO_GMINB
#define UNO_GMINB 1
#endif
#ifndef UNO_XMINB
#define UNO_XMINB 1
#endif

namespace uno {

// ============================================================================== x passes
// smem: tile 8M | stage (xfwd: p rows 8M; xinv: spectrum rows, then d and u rows 16M) | tw M | twp M+1
template <int M, bool INV>
__host__ __device__ constexpr int xsmem_bytes() {
  return (8 * M + (INV ? 16 : 8) * M + M + (M + 1)) * (int)sizeof(double2);
}

// F1 / standalone forward: real rows of length N1 = 2M -> half spectrum [kx][z][y].
template <int M, int MODE>
__global__ void __launch_bounds__(fft_threads(M), M == 128 ? UNO_XMINB : 1) xfwd_kernel(Ctx cx, const double* __restrict__ src, int bofs) {
  constexpr int T = fft_threads(M);
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  extern __shared__ double2 smem[];
  double2* tile = smem;
  double2* pbuf = smem + 8 * M;
  double2* tw = pbuf + 8 * M;
  double2* twp = tw + M;
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int bx = bofs + blockIdx.x;  // block of 8 rows (a z-chunk launch covers a contiguous range)
  const long long row0 = (long long)bx * 8;  // row = (comp, z, y) within the load
  const long long voff = (long long)load * g.c * g.n + row0 * g.N1;
  const double2* src2 = reinterpret_cast<const double2*>(src + voff);
  double2* r2 = reinterpret_cast<double2*>(cx.r + voff);
  const double2* p2 = reinterpret_cast<const double2*>(cx.p + voff);
  bool upd = false;
  double alpha = 0.0;
  if (MODE == CG) {
    upd = st->iters > 0;
    alpha = st->alpha;
  }
  // all global reads in flight at once (cp.async), rows land transposed+swizzled in the tile
#pragma unroll
  for (int i = 0; i < (8 * M + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < 8 * M) {
      cp_async16(&tile[tidx(e & (M - 1), e / M)], src2 + e);
      if (MODE == CG && upd) cp_async16(&pbuf[e], p2 + e);
    }
  }
  cp_commit();
  for (int i = t; i < M; i += T) tw[i] = cx.tw.x[i];
  for (int i = t; i <= M; i += T) twp[i] = cx.tw.xpost[i];
  cp_wait<0>();
  __syncthreads();
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < (8 * M + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < 8 * M) {
      const int ti = tidx(e & (M - 1), e / M);
      double2 v = tile[ti];
      if (MODE == CG && upd) {  // r <- r - alpha p   (Alg 2 l.11)
        const double2 pv = pbuf[e];
        v.x = fma(-alpha, pv.x, v.x);
        v.y = fma(-alpha, pv.y, v.y);
        r2[e] = v;
        tile[ti] = v;
      }
      mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
  }
  __syncthreads();
  fft_tile<M, false>(tile, tw);

  const int y0 = (int)(row0 % g.N2);
  const long long zc = row0 / g.N2;
  const int z = (int)(zc % g.P3);
  const int comp = (int)(zc / g.P3);
  double2* out = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * g.N2 + y0;
  const long long plane = (long long)g.P3 * g.N2;
#pragma unroll
  for (int i = 0; i < ((M / 2 + 1) * 8 + T - 1) / T; ++i) {
    const int it = t + i * T;
    if (it < (M / 2 + 1) * 8) {
      const int row = it & 7, k = it >> 3;
      const double2 a = tile[tidx(k, row)];
      const double2 b = cconj(tile[tidx((M - k) & (M - 1), row)]);
      const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
      const double2 O = mul_mi(make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y)));
      out[(long long)k * plane + row] = cadd(E, cmul(twp[k], O));
      if (k != M - k) out[(long long)(M - k) * plane + row] = cadd(cconj(E), cmul(twp[M - k], cconj(O)));
    }
  }
  if (MODE == CG) partial_write<true>(cx, RED_RNORM, load, bx, mx, red_sh);
}

// F1 for N1 = 256, register-direct: the complex FFT of length M = 128 (z_j = r_2j + i r_2j+1)
// as 8-point DFTs over n2 (j = n1 + 16 n2, thread = n1, 16 threads per row) -> twiddle
// w_128^{n1 k1} -> padded transpose -> 16-point DFT over n1 split between two threads
// (dft_half) -> X[k1 + 8 k2] to a swizzled row buffer -> R2C post-processing straight to the
// half spectrum.  r -= alpha p, ||r||_inf and the r write-back happen on the registers loaded.
constexpr int XR_RS = 8 * 17;             // transpose buffer per row (8 x 16, padded)
constexpr int XR_XS = 129;                // X row stride (odd in 16-byte units)
__device__ __forceinline__ int xr_swz(int k) { return k ^ (((k >> 3) & 1) << 2); }
template <int MODE>
__global__ void __launch_bounds__(128) xfwd256_kernel(Ctx cx, const double* __restrict__ src, int bofs) {
  constexpr int M = 128;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  __shared__ double2 tb[8 * XR_RS];
  __shared__ double2 xs[8 * XR_XS];
  __shared__ double2 tw[M];
  __shared__ double2 twp[M + 1];
  __shared__ double2 tw16[8];  // w_16^r = w_128^{8r}
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int r = t >> 4, l16 = t & 15;
  const int bx = bofs + blockIdx.x;
  const long long row0 = (long long)bx * 8;  // row = (comp, z, y)
  const long long voff = (long long)load * g.c * g.n + (row0 + r) * g.N1;
  const double2* s2 = reinterpret_cast<const double2*>(src + voff);
  double2 v[8];
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2) v[n2] = __ldcg(s2 + l16 + 16 * n2);
  double mx = 0.0;
  if (MODE == CG) {
    if (st->iters > 0) {  // r <- r - alpha p   (Alg 2 l.11)
      const double alpha = st->alpha;
      const double2* p2 = reinterpret_cast<const double2*>(cx.p + voff);
      double2* r2 = reinterpret_cast<double2*>(cx.r + voff);
      double2 pv[8];
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) pv[n2] = __ldcs(p2 + l16 + 16 * n2);
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) {
        v[n2].x = fma(-alpha, pv[n2].x, v[n2].x);
        v[n2].y = fma(-alpha, pv[n2].y, v[n2].y);
        __stcg(r2 + l16 + 16 * n2, v[n2]);
      }
    }
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) mx = fmax(mx, fmax(fabs(v[n2].x), fabs(v[n2].y)));
  }
  for (int i = t; i < M; i += 128) tw[i] = cx.tw.x[((i & 15) * (i >> 4)) & (M - 1)];  // [k1][n1]
  for (int i = t; i <= M; i += 128) twp[i] = cx.tw.xpost[i];
  if (t < 8) tw16[t] = cx.tw.x[8 * t];
  // ||r||_inf partial of the block: rides on this barrier (max is order-independent) — a block
  // reduce at the end kept every thread of these short-lived CTAs until the last store was issued:
  // 268.1 -> 260.7 us per launch at 256^3 x 3 loads
  if (MODE == CG) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) red_sh[t >> 5] = mx;
  }
  __syncthreads();
  if (MODE == CG && t == 0)
    red_partials(cx.sc, RED_RNORM, load)[bx] = fmax(fmax(red_sh[0], red_sh[1]), fmax(red_sh[2], red_sh[3]));
  // stage 1 (thread = n1): DFT8 over n2 -> k1, twiddle w_128^{n1 k1} (table [k1][n1])
  dft_reg<8, false>(v);
#pragma unroll
  for (int k1 = 1; k1 < 8; ++k1) v[k1] = cmul(v[k1], tw[k1 * 16 + l16]);
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) tb[r * XR_RS + k1 * 17 + l16] = v[k1];
  __syncthreads();
  // stage 2 (thread = (k1, h)): half of DFT16 over n1 -> k2 = 2m + h ; X[k1 + 8 k2]
  {
    const int k1 = l16 >> 1, h = l16 & 1;
    double2 a[16], o[8];
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) a[n1] = tb[r * XR_RS + k1 * 17 + n1];
    dft_half<16, false>(a, h, tw16, o);
#pragma unroll
    for (int m = 0; m < 8; ++m) xs[r * XR_XS + xr_swz(k1 + 8 * (2 * m + h))] = o[m];
  }
  __syncthreads();
  // R2C post-processing: bins k and M - k of row c
  const int y0 = (int)(row0 % g.N2);
  const long long zc = row0 / g.N2;
  const int z = (int)(zc % g.P3);
  const int comp = (int)(zc / g.P3);
  double2* out = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * g.N2 + y0;
  const long long plane = (long long)g.P3 * g.N2;
  for (int it = t; it < (M / 2 + 1) * 8; it += 128) {
    const int c = it & 7, k = it >> 3;
    const double2 a = xs[c * XR_XS + xr_swz(k)];
    const double2 b = cconj(xs[c * XR_XS + xr_swz((M - k) & (M - 1))]);
    const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
    const double2 O = mul_mi(make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y)));
    __stcg(out + (long long)k * plane + c, cadd(E, cmul(twp[k], O)));
    if (k != M - k) __stcg(out + (long long)(M - k) * plane + c, cadd(cconj(E), cmul(twp[M - k], cconj(O))));
  }
}

// F1 for N1 = 512 (config 4), register-direct: the complex FFT of length M = 256 (z_j = r_2j +
// i r_2j+1) as DFT16 over n2 (j = n1 + 16 n2, thread = n1, 16 threads per row) -> twiddle
// w_256^{n1 k1} -> padded transpose -> DFT16 over n1 (thread = k1) -> X[k1 + 16 k2] into a row
// buffer (stride 257, odd: conflict-free both ways; it reuses the transpose buffer) -> R2C
// post-processing straight to the half spectrum.  CG: r -= alpha p, ||r||_inf, r write-back on
// the loaded registers, as in xfwd256_kernel.
constexpr int X5_RS = 16 * 17, X5_XS = 257;
template <int MODE>
__global__ void __launch_bounds__(128) xfwd512_kernel(Ctx cx, const double* __restrict__ src, int bofs) {
  constexpr int M = 256;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  __shared__ double2 tb[8 * X5_RS];  // transpose buffer, then the X rows (8 x 257 <= 8 x 272)
  __shared__ double2 tw[M];
  __shared__ double2 twp[M + 1];
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int r = t >> 4, l16 = t & 15;
  const int bx = bofs + blockIdx.x;
  const long long row0 = (long long)bx * 8;  // row = (comp, z, y)
  const long long voff = (long long)load * g.c * g.n + (row0 + r) * g.N1;
  const double2* s2 = reinterpret_cast<const double2*>(src + voff);
  double2 v[16];
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) v[n2] = __ldcg(s2 + l16 + 16 * n2);
  double mx = 0.0;
  if (MODE == CG) {
    if (st->iters > 0) {  // r <- r - alpha p   (Alg 2 l.11)
      const double alpha = st->alpha;
      const double2* p2 = reinterpret_cast<const double2*>(cx.p + voff);
      double2* r2 = reinterpret_cast<double2*>(cx.r + voff);
#pragma unroll
      for (int h8 = 0; h8 < 16; h8 += 8) {
        double2 pv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pv[i] = __ldcs(p2 + l16 + 16 * (h8 + i));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[h8 + i].x = fma(-alpha, pv[i].x, v[h8 + i].x);
          v[h8 + i].y = fma(-alpha, pv[i].y, v[h8 + i].y);
          __stcg(r2 + l16 + 16 * (h8 + i), v[h8 + i]);
        }
      }
    }
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) mx = fmax(mx, fmax(fabs(v[n2].x), fabs(v[n2].y)));
  }
  for (int i = t; i < M; i += 128) tw[i] = cx.tw.x[((i & 15) * (i >> 4)) & (M - 1)];  // [k1][n1]
  for (int i = t; i <= M; i += 128) twp[i] = cx.tw.xpost[i];
  if (MODE == CG) {  // ||r||_inf partial of the block on this barrier (see xfwd256_kernel)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) red_sh[t >> 5] = mx;
  }
  __syncthreads();
  if (MODE == CG && t == 0)
    red_partials(cx.sc, RED_RNORM, load)[bx] = fmax(fmax(red_sh[0], red_sh[1]), fmax(red_sh[2], red_sh[3]));
  dft_reg<16, false>(v);  // thread = n1: over n2 -> k1
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], tw[k1 * 16 + l16]);
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) tb[r * X5_RS + k1 * 17 + l16] = v[k1];
  __syncthreads();
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) v[n1] = tb[r * X5_RS + l16 * 17 + n1];
  dft_reg<16, false>(v);  // thread = k1: v[k2] = X[k1 + 16 k2]
  __syncthreads();        // every transpose read done: the buffer becomes the X rows
  double2* xs = tb;
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) xs[r * X5_XS + l16 + 16 * k2] = v[k2];
  __syncthreads();
  // R2C post-processing: bins k and M - k of row c
  const int y0 = (int)(row0 % g.N2);
  const long long zc = row0 / g.N2;
  const int z = (int)(zc % g.P3);
  const int comp = (int)(zc / g.P3);
  double2* out = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * g.N2 + y0;
  const long long plane = (long long)g.P3 * g.N2;
  for (int it = t; it < (M / 2 + 1) * 8; it += 128) {
    const int c = it & 7, k = it >> 3;
    const double2 a = xs[c * X5_XS + k];
    const double2 b = cconj(xs[c * X5_XS + ((M - k) & (M - 1))]);
    const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
    const double2 O = mul_mi(make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y)));
    __stcg(out + (long long)k * plane + c, cadd(E, cmul(twp[k], O)));
    if (k != M - k) __stcg(out + (long long)(M - k) * plane + c, cadd(cconj(E), cmul(twp[M - k], cconj(O))));
  }
}

// F5 / standalone inverse: half spectrum -> real rows; CG epilogue d = s + beta d, u += alpha d_old.
template <int M, int MODE>
__global__ void __launch_bounds__(fft_threads(M)) xinv_kernel(Ctx cx, double* __restrict__ dst, int bofs) {
  constexpr int T = fft_threads(M);
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  extern __shared__ double2 smem[];
  double2* tile = smem;
  double2* stage = smem + 8 * M;   // [M+1][8] spectrum rows, later d rows [8M] | u rows [8M]
  double2* tw = stage + 16 * M;
  double2* twp = tw + M;
  const int t = threadIdx.x;
  const long long row0 = (long long)(bofs + blockIdx.x) * 8;
  const int y0 = (int)(row0 % g.N2);
  const long long zc = row0 / g.N2;
  const int z = (int)(zc % g.P3);
  const int comp = (int)(zc / g.P3);
  const double2* in = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * g.N2 + y0;
  const long long plane = (long long)g.P3 * g.N2;
#pragma unroll
  for (int i = 0; i < ((M + 1) * 8 + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < (M + 1) * 8) cp_async16(&stage[e], in + (long long)(e >> 3) * plane + (e & 7));
  }
  cp_commit();
  for (int i = t; i < M; i += T) tw[i] = cx.tw.x[i];
  for (int i = t; i <= M; i += T) twp[i] = cx.tw.xpost[i];
  cp_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ((M / 2 + 1) * 8 + T - 1) / T; ++i) {
    const int it = t + i * T;
    if (it < (M / 2 + 1) * 8) {
      const int row = it & 7, k = it >> 3;
      if (k == 0) {
        const double X0 = stage[row].x, XM = stage[M * 8 + row].x;
        tile[tidx(0, row)] = make_double2(X0 + XM, X0 - XM);
      } else {
        const double2 a = stage[k * 8 + row];
        const double2 bm = stage[(M - k) * 8 + row];
        const double2 b = cconj(bm);
        const double2 E = cadd(a, b);
        const double2 O = cmul(csub(a, b), cconj(twp[k]));
        tile[tidx(k, row)] = cadd(E, mul_pi(O));
        if (k != M - k) {
          const double2 a2 = bm, b2 = cconj(a);
          const double2 E2 = cadd(a2, b2);
          const double2 O2 = cmul(csub(a2, b2), cconj(twp[M - k]));
          tile[tidx(M - k, row)] = cadd(E2, mul_pi(O2));
        }
      }
    }
  }
  __syncthreads();
  const long long voff = (long long)load * g.c * g.n + row0 * g.N1;
  const int it0 = MODE == CG ? st->iters : 0;
  // paired u updates (cx.d2): direction j = it0 is written to (j & 1) ? d2 : d and d_{j-1} read
  // from the other buffer; u is touched only for even j >= 2, where u += alpha_{j-2} d_{j-2} +
  // alpha_{j-1} d_{j-1} (d_{j-2} = the rows about to be overwritten): 28 instead of 32 B/DOF of
  // vector traffic on average.  Without d2: u += alpha_{j-1} d_{j-1} every iteration.
  const bool pair = MODE == CG && cx.d2 != nullptr;
  double* dnew = pair && (it0 & 1) ? cx.d2 : cx.d;
  const double* dold = pair && !(it0 & 1) ? cx.d2 : cx.d;
  const bool do_u = pair ? (it0 >= 2 && !(it0 & 1)) : it0 > 0;
  if (MODE == CG) {  // d_old and u rows land while the inverse FFT runs
    const double2* d2g = reinterpret_cast<const double2*>(dold + voff);
    const double2* u2g = reinterpret_cast<const double2*>(cx.u + voff);
    if (it0 > 0) {
#pragma unroll
      for (int i = 0; i < (8 * M + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < 8 * M) {
          cp_async16(&stage[e], d2g + e);
          if (do_u) cp_async16(&stage[8 * M + e], u2g + e);
        }
      }
      if (pair && do_u) {  // d_{j-2} rows: read in the epilogue straight from L2
        const char* pb = reinterpret_cast<const char*>(dnew + voff);
        for (int o = t * 128; o < 8 * M * 16; o += T * 128) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pb + o));
      }
    }
    cp_commit();
    if (pair && do_u && blockIdx.x == 0 && t == 0) st->u_done = it0;  // terms 0 .. it0-1 are in u
  }
  fft_tile<M, true>(tile, tw);
  if (MODE != CG) {
    double2* o2 = reinterpret_cast<double2*>(dst + voff);
#pragma unroll
    for (int i = 0; i < (8 * M + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < 8 * M) o2[e] = tile[tidx(e & (M - 1), e / M)];
    }
  } else {
    cp_wait<0>();
    __syncthreads();
    double2* d2 = reinterpret_cast<double2*>(dnew + voff);
    double2* u2 = reinterpret_cast<double2*>(cx.u + voff);
    const double beta = st->beta, alpha = st->alpha, alpha2 = st->alpha_prev;
#pragma unroll
    for (int i = 0; i < (8 * M + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < 8 * M) {
        const double2 s = tile[tidx(e & (M - 1), e / M)];
        if (it0 == 0) {
          d2[e] = s;  // d = s + (gamma1/gamma0) * 0   (Alg 2 l.2, l.8)
        } else {
          const double2 dold = stage[e];
          if (do_u) {  // deferred u += [alpha_{m-2} d_{m-2} +] alpha_{m-1} d_{m-1}  (Alg 2 l.12)
            double2 uu = stage[8 * M + e];
            if (pair) {
              const double2 dm2 = __ldcg(d2 + e);
              uu.x = fma(alpha2, dm2.x, uu.x);
              uu.y = fma(alpha2, dm2.y, uu.y);
            }
            uu.x = fma(alpha, dold.x, uu.x);
            uu.y = fma(alpha, dold.y, uu.y);
            u2[e] = uu;
          }
          d2[e] = make_double2(fma(beta, dold.x, s.x), fma(beta, dold.y, s.y));
        }
      }
    }
  }
}

// F5 for N1 = 512 (config 4), register-direct: the 257 half-spectrum bins of 8 rows land in
// shared memory (row-major, stride 257: conflict-free); thread (row, k1) forms its 16 C2R
// inputs Z[k1 + 16 k2] = (X_k + conj X_{M-k}) + i (X_k - conj X_{M-k}) conj(w^k_post) directly,
// runs the inverse four-step (DFT16 over k2 -> twiddle conj w_256^{n1 k1} -> transpose -> DFT16
// over k1) and holds x[n1 + 16 n2] = (s_2j, s_2j+1) in registers for the CG epilogue
// d = s + beta d_old, u += alpha d_old (Alg 2 l.8, l.12).  Same arithmetic as xinv_kernel<256>.
constexpr int XI5_SS = 257, XI5_RS = 16 * 17;
template <int MODE>
__global__ void __launch_bounds__(128) xinv512_kernel(Ctx cx, double* __restrict__ dst, int bofs) {
  constexpr int M = 256;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  __shared__ double2 sb[8 * XI5_RS];  // spectrum rows [8][257], then the transpose buffer [8][16][17]
  __shared__ double2 tw[M];
  __shared__ double2 twp[M + 1];
  const int t = threadIdx.x;
  const int r = t >> 4, l16 = t & 15;
  const long long row0 = (long long)(bofs + blockIdx.x) * 8;
  const int y0 = (int)(row0 % g.N2);
  const long long zc = row0 / g.N2;
  const int z = (int)(zc % g.P3);
  const int comp = (int)(zc / g.P3);
  const double2* in = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * g.N2 + y0;
  const long long plane = (long long)g.P3 * g.N2;
#pragma unroll
  for (int i = 0; i < ((M + 1) * 8 + 127) / 128; ++i) {  // bin k of row c -> sb[c][k]
    const int e = t + i * 128;
    if (e < (M + 1) * 8) cp_async16(&sb[(e & 7) * XI5_SS + (e >> 3)], in + (long long)(e >> 3) * plane + (e & 7));
  }
  cp_commit();
  // paired u updates (cx.d2; see xinv_kernel): direction j = iters goes to (j & 1) ? d2 : d, u is
  // updated with two terms for even j >= 2 only
  const int it0 = MODE == CG ? st->iters : 0;
  const bool pair = MODE == CG && cx.d2 != nullptr;
  double* dnew = pair && (it0 & 1) ? cx.d2 : cx.d;
  double* dold = pair && !(it0 & 1) ? cx.d2 : cx.d;
  const bool do_u = pair ? (it0 >= 2 && !(it0 & 1)) : it0 > 0;
  if (MODE == CG && it0 > 0) {  // the 8 rows of d_old (and u, d_{j-2}) into L2 for the epilogue
    const long long o = (long long)load * g.c * g.n + row0 * g.N1;
    const char* db = reinterpret_cast<const char*>(dold + o);
    const char* ub = reinterpret_cast<const char*>(cx.u + o);
    const char* nb = reinterpret_cast<const char*>(dnew + o);
    for (int i = t; i < 8 * 512 * 8 / 128; i += 128) {
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(db + 128LL * i));
      if (do_u) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(ub + 128LL * i));
      if (pair && do_u) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(nb + 128LL * i));
    }
    if (pair && do_u && blockIdx.x == 0 && t == 0) st->u_done = it0;  // terms 0 .. it0-1 are in u
  }
  for (int i = t; i < M; i += 128) tw[i] = cx.tw.x[((i & 15) * (i >> 4)) & (M - 1)];  // [k1][n1]
  for (int i = t; i <= M; i += 128) twp[i] = cx.tw.xpost[i];
  cp_wait<0>();
  __syncthreads();
  double2 v[16];
  {
    const double2* row = sb + r * XI5_SS;
    const int k1 = l16;
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const int k = k1 + 16 * k2;
      if (k == 0) {
        const double X0 = row[0].x, XM = row[M].x;
        v[0] = make_double2(X0 + XM, X0 - XM);
      } else {
        const double2 a = row[k], b = cconj(row[M - k]);
        const double2 E = cadd(a, b);
        const double2 O = cmul(csub(a, b), cconj(twp[k]));
        v[k2] = cadd(E, mul_pi(O));
      }
    }
  }
  dft_reg<16, true>(v);  // thread = k1: inverse over k2 -> n1
#pragma unroll
  for (int n1 = 1; n1 < 16; ++n1) v[n1] = cmul(v[n1], cconj(tw[n1 * 16 + l16]));
  __syncthreads();  // every read of the spectrum rows done: sb becomes the transpose buffer
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) sb[r * XI5_RS + n1 * 17 + l16] = v[n1];
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) v[k1] = sb[r * XI5_RS + l16 * 17 + k1];
  dft_reg<16, true>(v);  // thread = n1: inverse over k1 -> n2 ; v[n2] = x[n1 + 16 n2]
  const long long voff = (long long)load * g.c * g.n + (row0 + r) * g.N1;
  if (MODE != CG) {
    double2* o2 = reinterpret_cast<double2*>(dst + voff);
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) __stcg(o2 + l16 + 16 * n2, v[n2]);
  } else {
    double2* d2 = reinterpret_cast<double2*>(dnew + voff);
    const double2* o2 = reinterpret_cast<const double2*>(dold + voff);
    double2* u2 = reinterpret_cast<double2*>(cx.u + voff);
    if (it0 == 0) {
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2) __stcg(d2 + l16 + 16 * n2, v[n2]);  // d = s (Alg 2 l.2, l.8)
    } else {
      const double beta = st->beta, alpha = st->alpha, alpha2 = st->alpha_prev;
#pragma unroll
      for (int h8 = 0; h8 < 16; h8 += 8) {
        double2 dold8[8], uu[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          dold8[i] = __ldcs(o2 + l16 + 16 * (h8 + i));
          if (do_u) uu[i] = __ldcs(u2 + l16 + 16 * (h8 + i));
        }
        if (do_u && pair) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // + alpha_{m-2} d_{m-2} (the rows about to be overwritten)
            const double2 dm2 = __ldcs(d2 + l16 + 16 * (h8 + i));
            uu[i].x = fma(alpha2, dm2.x, uu[i].x);
            uu[i].y = fma(alpha2, dm2.y, uu[i].y);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (do_u) {
            uu[i].x = fma(alpha, dold8[i].x, uu[i].x);  // deferred u += alpha_{m-1} d_{m-1} (l.12)
            uu[i].y = fma(alpha, dold8[i].y, uu[i].y);
            __stcg(u2 + l16 + 16 * (h8 + i), uu[i]);
          }
          const double2 s = v[h8 + i];
          __stcg(d2 + l16 + 16 * (h8 + i), make_double2(fma(beta, dold8[i].x, s.x), fma(beta, dold8[i].y, s.y)));
        }
      }
    }
  }
}

// ============================================================================== y pass (3D)
template <int L>
__host__ __device__ constexpr int ysmem_bytes() {
  return (8 * L + L) * (int)sizeof(double2);
}

template <int L, bool INV, int MODE>
__global__ void __launch_bounds__(fft_threads(L), L == 256 ? UNO_YMINB : 1) ypass_kernel(Ctx cx, int z0, int zc) {
  constexpr int T = fft_threads(L);
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tile = smem;
  double2* tw = smem + 8 * L;
  const int t = threadIdx.x;
  const long long nrows = (long long)g.c * g.H1 * g.P3;
  long long row0 = (long long)blockIdx.x * 8;  // row = (comp, kx, z)
  if (zc > 0) {  // z-chunk [z0, z0+zc) of every (comp, kx) plane (zc, z0 multiples of 8)
    const int nb = zc >> 3;
    const int q = blockIdx.x / nb;
    row0 = (long long)q * g.P3 + z0 + (blockIdx.x - q * nb) * 8;
  }
  double2* base = cx.spec + (long long)load * g.c * g.nspec + row0 * L;
  const bool full = row0 + 8 <= nrows;
#pragma unroll
  for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < 8 * L) {
      const int row = e / L, j = e & (L - 1);
      if (full || row0 + row < nrows)
        cp_async16(&tile[tidx(j, row)], base + e);
      else
        tile[tidx(j, row)] = make_double2(0.0, 0.0);
    }
  }
  cp_commit();
  for (int i = t; i < L; i += T) tw[i] = cx.tw.y[i];
  cp_wait<0>();
  __syncthreads();
  fft_tile<L, INV>(tile, tw);
#pragma unroll
  for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < 8 * L) {
      const int row = e / L, j = e & (L - 1);
      if (full || row0 + row < nrows) base[e] = tile[tidx(j, row)];
    }
  }
}

// y pass for N2 = 256, register-direct four-step (256 = 16 x 16, y = n1 + 16 n2,
// k = k1 + 16 k2): each of 16 threads per row loads its 16 elements n1 + 16 n2 straight into
// registers (coalesced across n1), does DFT16 over n2 and the twiddle w_256^{n1 k1}, one padded
// shared-memory transpose, then DFT16 over n1 and stores X[k1 + 16 k2] straight from
// registers.  One shared-memory round trip per element instead of four.
constexpr int YR_R = 16, YR_ROWS = 8, YR_RS = YR_R * (YR_R + 1);
template <bool INV, int MODE, bool PEER = false>
__global__ void __launch_bounds__(YR_ROWS * YR_R) ypass256_kernel(Ctx cx, int z0, int zc) {
  constexpr int L = 256;
  const Geo g = cx.g;
#if UNO_SERP
  // load fastest in the launch order (the hardware issues CTAs x-fastest): the row blocks of all load
  // cases advance together through the k_x planes, so the tail this pass leaves in L2 holds the last
  // planes of every load — where the reversed G pass starts (and where the inverse y pass follows it)
  const unsigned lin = blockIdx.y * gridDim.x + blockIdx.x;
  const int load = (int)(lin % gridDim.y);
  const unsigned bxl = lin / gridDim.y;
#else
  const int load = blockIdx.y;
  const unsigned bxl = blockIdx.x;
#endif
  if (MODE == CG && !cx.st[load].active) return;
  __shared__ double2 buf[YR_ROWS * YR_RS];
#if !UNO_TWLDG_256
  __shared__ double2 tw[L];
#endif
  const int t = threadIdx.x;
  const int r = t >> 4, lane16 = t & 15;
  const long long nrows = (long long)g.c * g.H1 * g.P3;
  long long row0 = (long long)bxl * YR_ROWS;  // row = (comp, kx, z)
  if (zc > 0) {
    const int nb = zc >> 3;
    const int q = bxl / nb;
    row0 = (long long)q * g.P3 + z0 + (bxl - q * nb) * 8;
  }
  const bool ok = row0 + r < nrows;
  double2* rowp = cx.spec + (long long)load * g.c * g.nspec + (row0 + r) * L;
  double2 v[YR_R];
  if (ok) {
#pragma unroll
    for (int n2 = 0; n2 < YR_R; ++n2) v[n2] = __ldcg(rowp + lane16 + YR_R * n2);
  }
  // twiddle table tw[k1][n1] = w_256^{n1 k1}: a quarter-warp (8 consecutive n1) reads 8
  // consecutive entries (conflict-free)
#if !UNO_TWLDG_256
  for (int i = t; i < L; i += YR_ROWS * YR_R) tw[i] = cx.tw.y[((i & 15) * (i >> 4)) & (L - 1)];
  __syncthreads();
#endif
  // stage 1 (thread = n1): DFT16 over n2 -> k1, twiddle w_256^{n1 k1}
  dft_reg<YR_R, INV>(v);
  {
    const int n1 = lane16;
#pragma unroll
    for (int k1 = 1; k1 < YR_R; ++k1) {
#if UNO_TWLDG_256
      // straight from the 4 KB table through L1: no staging copy and no barrier before stage 1
      const double2 w = __ldg(cx.tw.y + ((k1 * n1) & (L - 1)));
#else
      const double2 w = tw[k1 * YR_R + n1];
#endif
      v[k1] = cmul(v[k1], INV ? cconj(w) : w);
    }
#pragma unroll
    for (int k1 = 0; k1 < YR_R; ++k1) buf[r * YR_RS + k1 * (YR_R + 1) + n1] = v[k1];
  }
  __syncthreads();
  // stage 2 (thread = k1): DFT16 over n1 -> k2 ; X[k1 + 16 k2]
  {
    const int k1 = lane16;
#pragma unroll
    for (int n1 = 0; n1 < YR_R; ++n1) v[n1] = buf[r * YR_RS + k1 * (YR_R + 1) + n1];
    dft_reg<YR_R, INV>(v);
    if (ok) {
      if constexpr (PEER) {  // slab: the all-to-all block of each bin goes straight to its owner
        const long long grow = (long long)load * nrows + row0 + r;
        const int yc = cx.peer_yc;
#pragma unroll
        for (int k2 = 0; k2 < YR_R; ++k2) {
          const int k = k1 + YR_R * k2;
          __stcg(cx.peer[k / yc] + cx.peer_off + grow * yc + (k & (yc - 1)), v[k2]);
        }
      } else {
#pragma unroll
        for (int k2 = 0; k2 < YR_R; ++k2) __stcg(rowp + k1 + YR_R * k2, v[k2]);
      }
    }
  }
  if constexpr (PEER) __threadfence_system();
}


// y pass for N2 = 512: 512 = 32 x 16 (y = n1 + 32 n2, k = k1 + 16 k2).  32 threads per row: each
// loads 16 elements, DFT16 over n2, twiddle w_512^{n1 k1}, padded transpose; then the 32-point
// DFTs over n1 (one per k1) are split between thread pairs (dft_half, outputs k2 = 2m + h) and
// stored straight from registers.  4 rows per 128-thread CTA.
constexpr int Y5_ROWS = 4, Y5_RS = 16 * 33;
template <bool INV, int MODE, bool PEER = false>
__global__ void __launch_bounds__(128) ypass512_kernel(Ctx cx, int z0, int zc) {
  constexpr int L = 512;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  __shared__ double2 buf[Y5_ROWS * Y5_RS];
#if !UNO_TWLDG_512
  __shared__ double2 tw[16 * 32];  // [k1][n1] = w_512^{n1 k1}
#endif
  __shared__ double2 tw32[16];     // w_32^r
  const int t = threadIdx.x;
  const int r = t >> 5, l32 = t & 31;
  const long long nrows = (long long)g.c * g.H1 * g.P3;
  long long row0 = (long long)blockIdx.x * Y5_ROWS;
  if (zc > 0) {
    const int nb = zc / Y5_ROWS;
    const int q = blockIdx.x / nb;
    row0 = (long long)q * g.P3 + z0 + (blockIdx.x - q * nb) * Y5_ROWS;
  }
  const bool ok = row0 + r < nrows;
  double2* rowp = cx.spec + (long long)load * g.c * g.nspec + (row0 + r) * L;
  double2 v[16];
  if (ok) {
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) v[n2] = __ldcg(rowp + l32 + 32 * n2);
  }
#if !UNO_TWLDG_512
  for (int i = t; i < 16 * 32; i += 128) tw[i] = cx.tw.y[((i & 31) * (i >> 5)) & (L - 1)];
#endif
  if (t < 16) tw32[t] = cx.tw.y[16 * t];
#if !UNO_TWLDG_512
  __syncthreads();
#endif
  dft_reg<16, INV>(v);  // thread = n1: over n2 -> k1
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) {
#if UNO_TWLDG_512
    const double2 w = __ldg(cx.tw.y + ((k1 * l32) & (L - 1)));  // 8 KB table through L1 (see ypass256_kernel)
#else
    const double2 w = tw[k1 * 32 + l32];
#endif
    v[k1] = cmul(v[k1], INV ? cconj(w) : w);
  }
  double2* Tr = buf + r * Y5_RS;
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) Tr[k1 * 33 + l32] = v[k1];
  __syncthreads();
  {
    const int k1 = l32 >> 1, h = l32 & 1;
    double2 a[32], o[16];
#pragma unroll
    for (int n1 = 0; n1 < 32; ++n1) a[n1] = Tr[k1 * 33 + n1];
    dft_half<32, INV>(a, h, tw32, o);
    if (ok) {
      if constexpr (PEER) {  // slab: each bin straight to the owner of its k_y chunk
        const long long grow = (long long)load * nrows + row0 + r;
        const int yc = cx.peer_yc;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const int k = k1 + 16 * (2 * m + h);
          __stcg(cx.peer[k / yc] + cx.peer_off + grow * yc + (k & (yc - 1)), o[m]);
        }
      } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) __stcg(rowp + k1 + 16 * (2 * m + h), o[m]);
      }
    }
  }
  if constexpr (PEER) __threadfence_system();
}

int launch_ypass_peer(const Ctx& cx, cudaStream_t s) {
  const Geo& g = cx.g;
  const long long nrows = (long long)g.c * g.H1 * g.P3;
  if (g.N2 == 256) {
    const dim3 grid((unsigned)((nrows + YR_ROWS - 1) / YR_ROWS), g.nrhs);
    ypass256_kernel<false, CG, true><<<grid, YR_ROWS * YR_R, 0, s>>>(cx, 0, 0);
    return 1;
  }
  if (g.N2 == 512) {
    const dim3 grid((unsigned)((nrows + Y5_ROWS - 1) / Y5_ROWS), g.nrhs);
    ypass512_kernel<false, CG, true><<<grid, 128, 0, s>>>(cx, 0, 0);
    return 1;
  }
  return -1;
}

template <int L, int NC>
__host__ __device__ constexpr int gsmem_tile_bytes() {
  return (NC * 8 * L + L) * (int)sizeof(double2);
}
// symbol entries of the tile's bins are staged in smem too when they fit
template <int L, int NC>
__host__ __device__ constexpr bool gstaged() {
  return gsmem_tile_bytes<L, NC>() + 8 * L * (NC == 1 ? 1 : (NC == 2 ? 3 : 6)) * (int)sizeof(double) <= 200 * 1024;
}
template <int L, int NC>
__host__ __device__ constexpr int gsmem_bytes() {
  return gsmem_tile_bytes<L, NC>() + (gstaged<L, NC>() ? 8 * L * (NC == 1 ? 1 : (NC == 2 ? 3 : 6)) * (int)sizeof(double) : 0);
}

// 3D G pass: sequences along z (stride N2), tile = 8 consecutive y of one kx plane.
template <int L, int NC, int MODE, bool PEER = false>
__global__ void __launch_bounds__(fft_threads(L), L == 256 ? UNO_GMINB : 1) gpass_z_kernel(Ctx cx) {
  constexpr int T = fft_threads(L);
  constexpr int NCC = NC == 1 ? 1 : (NC == 2 ? 3 : 6);  // unique symbol entries per bin
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tiles[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) tiles[q] = smem + q * 8 * L;
  double2* tw = smem + NC * 8 * L;
  double* gs = reinterpret_cast<double*>(tw + L);  // [NCC][8L] symbol entries of the tile's bins
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int ntile_y = g.N2 >> 3;
  const int kx = blockIdx.x / ntile_y;
  const int y0 = (blockIdx.x - kx * ntile_y) * 8;
  const long long boff = (long long)kx * g.N3 * g.N2 + y0;
  constexpr bool STG = gstaged<L, NC>() && MODE != FWDZ;
  // unstaged symbol (L = 512, c = 3: one CTA per SM): one copy group per component, so the forward
  // stages of component 0 run while 1 and 2 land, and each component is stored as soon as its
  // inverse is done (load / compute / store overlap inside the CTA)
  constexpr bool PIPE = !STG && NC == 3 && MODE != FWDZ && gconv_fusable(L) && NC * plan_radix(L, plan_stages(L) - 1) <= 32;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const double2* base = cx.spec + ((long long)load * g.c + q) * g.nspec + boff;
#pragma unroll
    for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < 8 * L) cp_async16(&tiles[q][tidx(e >> 3, e & 7)], base + (long long)(e >> 3) * g.N2 + (e & 7));
    }
    if (PIPE) cp_commit();
  }
  if constexpr (!STG && MODE != FWDZ) {
    // symbol too large to stage with the tile (L = 512, c = 3): pull its rows (8 bins, 64 bytes
    // each) into L2 now so the reads inside the fused butterfly hit L2 rather than DRAM
    for (int r = t; r < NCC * L; r += T) {
      const int ent = r / L, kz = r - ent * L;
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(cx.gtab + ent * g.nspec + boff + (long long)kz * g.N2));
    }
  }
  if (STG) {
#pragma unroll
    for (int q = 0; q < NCC; ++q) {
#pragma unroll
      for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < 8 * L) cp_async8(&gs[q * 8 * L + e], cx.gtab + q * g.nspec + boff + (long long)(e >> 3) * g.N2 + (e & 7));
      }
    }
  }
  if (!PIPE) cp_commit();
  for (int i = t; i < L; i += T) tw[i] = cx.tw.z[i];
  if (!PIPE) {
    cp_wait<0>();
    __syncthreads();
  }
  if constexpr (MODE == FWDZ) {  // forward z transform only (training features, train.cu)
#pragma unroll
    for (int q = 0; q < NC; ++q) fft_tile<L, false>(tiles[q], tw);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double2* base = cx.spec + ((long long)load * g.c + q) * g.nspec + boff;
#pragma unroll
      for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < 8 * L) base[(long long)(e >> 3) * g.N2 + (e & 7)] = tiles[q][tidx(e >> 3, e & 7)];
      }
    }
    return;
  }
  auto store_comp = [&](int q) {
    if constexpr (PEER) {  // slab: z plane zz belongs to rank zz / peer_z -> its receive buffer
      const long long lk = ((long long)load * g.c + q) * g.H1 + kx;
#pragma unroll
      for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < 8 * L) {
          const int zz = e >> 3, qd = zz / cx.peer_z, zq = zz - qd * cx.peer_z;
          cx.peer[qd][((cx.peer_rank * cx.peer_nlckx + lk) * cx.peer_z + zq) * g.N2 + y0 + (e & 7)] =
              tiles[q][tidx(zz, e & 7)];
        }
      }
    } else {
      double2* base = cx.spec + ((long long)load * g.c + q) * g.nspec + boff;
#pragma unroll
      for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < 8 * L) base[(long long)(e >> 3) * g.N2 + (e & 7)] = tiles[q][tidx(e >> 3, e & 7)];
      }
    }
  };
  const double w = parseval_w(kx, g.M);
  double part = 0.0;
  if constexpr (gconv_fusable(L) && NC * plan_radix(L, plan_stages(L) - 1) <= 32) {
    // symbol multiply fused into the middle butterfly (fft.cuh fft_gconv)
    auto mul = [&](int, int c, int kz, double2* x) {
      return STG ? gmul_vals<NC>(x, gs, 8 * L, (long long)kz * 8 + c, w)
                 : gmul_vals<NC>(x, cx.gtab, g.nspec, boff + (long long)kz * g.N2 + c, w);
    };
    if constexpr (PIPE) {
      auto pre = [&](int q) {
        if (q == 0) cp_wait<2>();
        else if (q == 1) cp_wait<1>();
        else cp_wait<0>();
        __syncthreads();
      };
      part = fft_gconv<L, 1, NC>(tiles, tw, mul, pre, store_comp);
    } else {
      part = fft_gconv<L, 1, NC>(tiles, tw, mul);
    }
  } else {
#pragma unroll
    for (int q = 0; q < NC; ++q) fft_tile<L, false>(tiles[q], tw);
#pragma unroll
    for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < 8 * L) {
        if (STG)
          part += gmul_bin<NC>(tiles, tidx(e >> 3, e & 7), gs, 8 * L, e, w);
        else
          part += gmul_bin<NC>(tiles, tidx(e >> 3, e & 7), cx.gtab, g.nspec, boff + (long long)(e >> 3) * g.N2 + (e & 7), w);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NC; ++q) fft_tile<L, true>(tiles[q], tw);
  }
  if constexpr (!PIPE) {
#pragma unroll
    for (int q = 0; q < NC; ++q) store_comp(q);
  }
  if constexpr (PEER) __threadfence_system();
  gamma_finish(cx, load, part, red_sh, MODE);
}

// Thermal G pass for N3 = 256, register-direct (same four-step as ypass256_kernel, along z):
// tile = 8 consecutive y columns of one kx plane, thread (c, l) with c the column, l = n1 in the
// loads / k1 after the first transpose.  Forward DFT16 (n2) -> twiddle -> transpose -> DFT16
// (n1) leaves the bins k1 + 16 k2 in registers, where s_hat = G_hat r_hat and the Parseval
// partial of gamma (Eq 46/49) are formed; the inverse mirrors the forward.  Column stride 273
// (odd in 16-byte units) keeps every quarter-warp access bank-conflict free.
constexpr int GR_CS = YR_R * (YR_R + 1) + 1;
#ifndef UNO_G256_MINB
#define UNO_G256_MINB 3  // resident CTAs per SM of the thermal 256-point G pass (A/B builds only)
#endif
template <int MODE>
__global__ void __launch_bounds__(8 * YR_R, UNO_G256_MINB) gpass256_kernel(Ctx cx) {  // smem: gpass256_smem
  constexpr int L = 256, R = YR_R, RP = R + 1;
  const Geo g = cx.g;
  // load fastest in the launch order: the nrhs CTAs of one tile read the same symbol rows back to
  // back, so the repeats are served from L2 (the table is read from HBM once per pass, not nrhs times)
  const int load = blockIdx.x % g.nrhs;
  const int tile = blockIdx.x / g.nrhs;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 gsm[];
  double2* buf = gsm;                                          // [8][GR_CS]
  double2* tw = buf + 8 * GR_CS;                               // [L]
  double* gs = reinterpret_cast<double*>(tw + L);              // [L][8] symbol of the tile's bins
  __shared__ double red_sh[32];
  const int t = threadIdx.x, c = t & 7, ln = t >> 3;
  const int ntile_y = g.N2 >> 3;
  const int kx = tile / ntile_y;
  const int y0 = (tile - kx * ntile_y) * 8;
  const long long boff = (long long)kx * g.N3 * g.N2 + y0;
  double2* col = cx.spec + (long long)load * g.nspec + boff + c;
  const long long zs = g.N2;
  // symbol of the tile lands in shared memory while the forward transform runs
#pragma unroll
  for (int i = 0; i < L * 8 / (2 * 8 * R); ++i) {  // 16-byte copies: 2 bins each
    const int e = 2 * (t + i * 8 * R);
    cp_async16(&gs[e], cx.gtab + boff + (long long)(e >> 3) * zs + (e & 7));
  }
  cp_commit();
  double2 v[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) v[n2] = __ldcg(col + (ln + R * n2) * zs);
  for (int i = t; i < L; i += 8 * R) tw[i] = cx.tw.z[i];
  __syncthreads();
  double2* bc = buf + c * GR_CS;
  dft_reg<R, false>(v);  // thread = n1: DFT over n2 -> k1
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) v[k1] = cmul(v[k1], tw[(ln * k1) & (L - 1)]);
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) bc[k1 * RP + ln] = v[k1];
  __syncthreads();
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = bc[ln * RP + n1];
  dft_reg<R, false>(v);  // thread = k1: v[k2] = r_hat(kz = k1 + 16 k2)
  const double w = parseval_w(kx, g.M);
  cp_wait<0>();
  __syncthreads();
  double part = 0.0;
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) part += gmul_vals<1>(&v[k2], gs + c, 0, (long long)(ln + R * k2) * 8, w);
  dft_reg<R, true>(v);  // inverse over k2 -> n1 (thread = k1)
#pragma unroll
  for (int n1 = 1; n1 < R; ++n1) v[n1] = cmul(v[n1], cconj(tw[(ln * n1) & (L - 1)]));
  __syncthreads();  // every stage-2 read of buf done
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) bc[n1 * RP + ln] = v[n1];
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) v[k1] = bc[ln * RP + k1];
  dft_reg<R, true>(v);  // thread = n1: inverse over k1 -> n2
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) __stcg(col + (ln + R * n2) * zs, v[n2]);
  partial_write<false>(cx, RED_GAMMA, load, tile, part, red_sh);
}

// Elastic G pass for N3 = 256 (c = 3), register-direct: tile = 4 consecutive y columns of one kx
// plane, all three components; thread (q, c, l) = component q, column c, l as in gpass256_kernel.
// After the forward four-step each thread holds r_hat_q at the bins k1 + 16 k2 of its column; the
// bins go to shared memory once so that thread q forms row q of the 3x3 block multiply
// s_hat_q = sum_p G_qp r_hat_p (Eq B7 entry order) and its share of the Parseval partial.  The
// (component, column) buffers use stride 274 (= 2 mod 8 in 16-byte units): a quarter warp (4
// columns x 2 l) hits 8 distinct bank groups.  2 CTAs/SM (106 KB of smem each).
constexpr int GE_COLS = 4, GE_CS = YR_R * (YR_R + 1) + 2;
constexpr int gpass256e_smem = (3 * GE_COLS * GE_CS + 256) * 16 + 6 * 256 * GE_COLS * 8;
template <int MODE>
__global__ void __launch_bounds__(3 * GE_COLS * YR_R, 2) gpass256e_kernel(Ctx cx) {
  constexpr int L = 256, R = YR_R, RP = R + 1;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 gsm[];
  double2* buf = gsm;                                  // [3][GE_COLS][GE_CS]
  double2* tw = buf + 3 * GE_COLS * GE_CS;             // [L]
  double* gs = reinterpret_cast<double*>(tw + L);      // [6][L][GE_COLS] symbol of the tile's bins
  __shared__ double red_sh[32];
  const int t = threadIdx.x, c = t & (GE_COLS - 1), ln = (t >> 2) & (R - 1), q = t >> 6;
  const int ntile_y = g.N2 / GE_COLS;
  const int kx = blockIdx.x / ntile_y;
  const int y0 = (blockIdx.x - kx * ntile_y) * GE_COLS;
  const long long boff = (long long)kx * g.N3 * g.N2 + y0;
  double2* col = cx.spec + ((long long)load * 3 + q) * g.nspec + boff + c;
  const long long zs = g.N2;
#pragma unroll
  for (int i = 0; i < 6 * L * GE_COLS / (2 * 3 * GE_COLS * R); ++i) {  // 16-byte copies: 2 bins each
    const int e = 2 * (t + i * 3 * GE_COLS * R);                     // e = (ent * L + kz) * 4 + cc
    const int ent = e / (L * GE_COLS), kz = (e / GE_COLS) & (L - 1), cc = e & (GE_COLS - 1);
    cp_async16(&gs[e], cx.gtab + ent * g.nspec + boff + (long long)kz * zs + cc);
  }
  cp_commit();
  double2 v[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) v[n2] = __ldcg(col + (ln + R * n2) * zs);
  for (int i = t; i < L; i += 3 * GE_COLS * R) tw[i] = cx.tw.z[i];
  __syncthreads();
  double2* bc = buf + (q * GE_COLS + c) * GE_CS;
  dft_reg<R, false>(v);  // thread = n1: DFT over n2 -> k1
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) v[k1] = cmul(v[k1], tw[(ln * k1) & (L - 1)]);
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) bc[k1 * RP + ln] = v[k1];
  __syncthreads();
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = bc[ln * RP + n1];
  dft_reg<R, false>(v);  // thread = k1: v[k2] = r_hat_q(kz = k1 + 16 k2)
  __syncthreads();       // every stage-2 read of buf done
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) bc[k2 * RP + ln] = v[k2];
  cp_wait<0>();
  __syncthreads();
  const double w = parseval_w(kx, g.M);
  // row q of the block in Eq B7 order (v1=G11 v2=G22 v3=G12 v4=G33 v5=G23 v6=G13): the own
  // component stays in registers, the other two (p1 = q+1, p2 = q+2 mod 3) come from smem
  const int p1 = q == 2 ? 0 : q + 1, p2 = q == 0 ? 2 : q - 1;
  const int eq = q == 0 ? 0 : (q == 1 ? 1 : 3);   // G_qq
  const int e1 = q == 0 ? 2 : (q == 1 ? 4 : 5);   // G_q,p1: G12, G23, G31
  const int e2 = q == 0 ? 5 : (q == 1 ? 2 : 4);   // G_q,p2: G13, G21, G32
  const double2* b1 = buf + (p1 * GE_COLS + c) * GE_CS;
  const double2* b2 = buf + (p2 * GE_COLS + c) * GE_CS;
  const double* gq = gs + eq * L * GE_COLS + c;
  const double* g1 = gs + e1 * L * GE_COLS + c;
  const double* g2 = gs + e2 * L * GE_COLS + c;
  double part = 0.0;
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) {
    const int kz = (ln + R * k2) * GE_COLS;
    const double2 X1 = b1[k2 * RP + ln], X2 = b2[k2 * RP + ln];
    const double a = gq[kz], b = g1[kz], cc = g2[kz];
    double2 Y;
    Y.x = fma(a, v[k2].x, fma(b, X1.x, cc * X2.x));
    Y.y = fma(a, v[k2].y, fma(b, X1.y, cc * X2.y));
    part = fma(w, fma(v[k2].x, Y.x, v[k2].y * Y.y), part);
    v[k2] = Y;
  }
  dft_reg<R, true>(v);  // inverse over k2 -> n1 (thread = k1)
#pragma unroll
  for (int n1 = 1; n1 < R; ++n1) v[n1] = cmul(v[n1], cconj(tw[(ln * n1) & (L - 1)]));
  __syncthreads();  // every multiply read of buf done
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) bc[n1 * RP + ln] = v[n1];
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) v[k1] = bc[ln * RP + k1];
  dft_reg<R, true>(v);  // thread = n1: inverse over k1 -> n2
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) __stcg(col + (ln + R * n2) * zs, v[n2]);
  gamma_finish(cx, load, part, red_sh, MODE);
}

// Thermal G pass for N3 = 512, register-direct four-step 512 = 32 x 16 along z (the z analogue of
// ypass512_kernel): tile = 4 consecutive y columns of one kx plane, thread (n1, c) = ((t >> 2) & 31,
// t & 3), so a warp loads 64-byte segments of 8 z rows.  Forward: DFT16 over n2 -> twiddle ->
// transpose -> DFT32 over n1 split between thread pairs (dft_half: thread h gets the bins
// k1 + 16 (2m + h)), where s_hat = G_hat r_hat and the Parseval partial are formed; the inverse
// mirrors it.  Every shared-memory pattern is conflict-free for a quarter warp (4 columns x 2
// threads): column buffers 546 apart (= 2 mod 8 in 16-byte units), k1-major rows of 34, and the
// final n1-major transpose swizzled as k1 ^ (n1 & 1).  (An elastic variant — 3 components x 4
// columns, 1 CTA/SM — measured 4.08 ms vs 3.67 ms for gpass_z_kernel at 512^3 and was dropped.)
constexpr int G5_CS = 546, G5_C = 4, G5_T = 32 * G5_C;
constexpr int gpass512_smem = (G5_C * G5_CS + 16 * 32 + 16) * 16 + 512 * G5_C * 8;
template <int MODE>
__global__ void __launch_bounds__(G5_T, 3) gpass512_kernel(Ctx cx) {
  constexpr int L = 512;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 gsm[];
  double2* buf = gsm;                                  // [G5_C][G5_CS]
  double2* tw = buf + G5_C * G5_CS;                    // [k1][n1] = w_512^{k1 n1}
  double2* tw32 = tw + 16 * 32;                        // w_32^r
  double* gs = reinterpret_cast<double*>(tw32 + 16);   // [L][G5_C] symbol of the tile's bins
  __shared__ double red_sh[32];
  const int t = threadIdx.x, c = t & (G5_C - 1), l32 = t >> 2;
  const int ntile_y = g.N2 / G5_C;
  const int kx = blockIdx.x / ntile_y;
  const int y0 = (blockIdx.x - kx * ntile_y) * G5_C;
  const long long boff = (long long)kx * g.N3 * g.N2 + y0;
  double2* col = cx.spec + (long long)load * g.nspec + boff + c;
  const long long zs = g.N2;
#pragma unroll
  for (int i0 = 0; i0 < L * G5_C / 2; i0 += G5_T) {  // 16-byte copies: 2 columns of one kz
    const int i = i0 + t;
    cp_async16(&gs[2 * i], cx.gtab + boff + (long long)(i >> 1) * zs + 2 * (i & 1));
  }
  cp_commit();
  double2 v[16];
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) v[n2] = __ldcg(col + (l32 + 32 * n2) * zs);
  for (int i = t; i < 16 * 32; i += G5_T) tw[i] = cx.tw.z[((i & 31) * (i >> 5)) & (L - 1)];
  if (t < 16) tw32[t] = cx.tw.z[16 * t];
  __syncthreads();
  double2* B = buf + c * G5_CS;
  dft_reg<16, false>(v);  // thread = n1: over n2 -> k1
#pragma unroll
  for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], tw[k1 * 32 + l32]);
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) B[k1 * 34 + l32] = v[k1];
  __syncthreads();
  const int k1 = l32 >> 1, h = l32 & 1;
  double2 o[16];
  {
    double2 a[32];
#pragma unroll
    for (int n1 = 0; n1 < 32; ++n1) a[n1] = B[k1 * 34 + n1];
    dft_half<32, false>(a, h, tw32, o);  // o[m] = r_hat(kz = k1 + 16 (2m + h))
  }
  const double w = parseval_w(kx, g.M);
  double part = 0.0;
  cp_wait<0>();
  __syncthreads();  // symbol landed; every stage-2 read of B done
#pragma unroll
  for (int m = 0; m < 16; ++m) part += gmul_vals<1>(&o[m], gs + c, 0, (long long)(k1 + 16 * (2 * m + h)) * G5_C, w);
#pragma unroll
  for (int m = 0; m < 16; ++m) B[k1 * 34 + 2 * m + h] = o[m];
  __syncthreads();
  {
    double2 a[32];
#pragma unroll
    for (int k2 = 0; k2 < 32; ++k2) a[k2] = B[k1 * 34 + k2];
    dft_half<32, true>(a, h, tw32, o);  // o[m] = x(n1 = 2m + h) of this k1
  }
  __syncthreads();  // every read of B done before the transposed writes
#pragma unroll
  for (int m = 0; m < 16; ++m) B[(2 * m + h) * 16 + (k1 ^ h)] = o[m];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = B[l32 * 16 + (j ^ (l32 & 1))];
#pragma unroll
  for (int j = 1; j < 16; ++j) v[j] = cmul(v[j], cconj(tw[j * 32 + l32]));
  dft_reg<16, true>(v);  // thread = n1: over k1 -> n2
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) __stcg(col + (l32 + 32 * n2) * zs, v[n2]);
  gamma_finish(cx, load, part, red_sh, MODE);
}

// G pass along y (contiguous rows): 2D grids (rows = kx) and the mixed-BC schedule (rows = (kx, m),
// m the DST-I mode along z, P3 planes); tile = 8 consecutive rows.
template <int L, int NC, int MODE>
__global__ void __launch_bounds__(fft_threads(L)) gpass_y2d_kernel(Ctx cx) {
  constexpr int T = fft_threads(L);
  constexpr int NCC = NC == 1 ? 1 : (NC == 2 ? 3 : 6);
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tiles[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) tiles[q] = smem + q * 8 * L;
  double2* tw = smem + NC * 8 * L;
  double* gs = reinterpret_cast<double*>(tw + L);  // [NCC][8 rows][L]
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int row0 = blockIdx.x * 8;
  const int nrows = g.H1 * g.P3;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const double2* base = cx.spec + ((long long)load * g.c + q) * g.nspec + (long long)row0 * L;
#pragma unroll
    for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < 8 * L) {
        const int row = e / L, j = e & (L - 1);
        if (row0 + row < nrows)
          cp_async16(&tiles[q][tidx(j, row)], base + e);
        else
          tiles[q][tidx(j, row)] = make_double2(0.0, 0.0);
      }
    }
  }
  constexpr bool STG = gstaged<L, NC>();
  if (STG) {
#pragma unroll
    for (int q = 0; q < NCC; ++q) {
#pragma unroll
      for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < 8 * L && row0 + e / L < nrows)
          cp_async8(&gs[q * 8 * L + e], cx.gtab + q * g.nspec + (long long)row0 * L + e);
      }
    }
  }
  cp_commit();
  for (int i = t; i < L; i += T) tw[i] = cx.tw.y[i];
  cp_wait<0>();
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NC; ++q) fft_tile<L, false>(tiles[q], tw);
  double part = 0.0;
#pragma unroll
  for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < 8 * L) {
      const int row = e & 7, j = e >> 3;
      const int rg = row0 + row;
      if (rg < nrows) {
        if (STG)
          part += gmul_bin<NC>(tiles, tidx(j, row), gs, 8 * L, row * L + j, parseval_w(rg / g.P3, g.M));
        else
          part += gmul_bin<NC>(tiles, tidx(j, row), cx.gtab, g.nspec, (long long)rg * L + j, parseval_w(rg / g.P3, g.M));
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NC; ++q) fft_tile<L, true>(tiles[q], tw);
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    double2* base = cx.spec + ((long long)load * g.c + q) * g.nspec + (long long)row0 * L;
#pragma unroll
    for (int i = 0; i < (8 * L + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < 8 * L) {
        const int row = e / L, j = e & (L - 1);
        if (row0 + row < nrows) base[e] = tiles[q][tidx(j, row)];
      }
    }
  }
  gamma_finish(cx, load, part, red_sh, MODE);
}

// ============================================================================== K apply
// Thermal 3D, cubic voxels.  For node i with octant elements o (conductivity k_o), the Q1
// element row (App. A1: h{1/3, 0, -1/12, -1/12}) gives
//   p_i = h/12 [ 5 d_i sum_o k_o + sum_{6 axis nbrs j} d_j (sum of k over the 4 octants
//         sharing edge ij) - sum_o k_o S_o ],   S_o = sum of the 8 corner values of o.
// CTA = TX x 8 nodes marching over ZC z-planes (2.5D blocking).  Node planes of d stream
// through a 7-deep shared-memory ring with cp.async (LDGSTS) issued 3 planes ahead, so HBM
// latency overlaps the arithmetic.  Each thread reads the 3x3 neighbourhood of plane k+1,
// forms the four element box sums of that plane in registers and carries every
// layer-k quantity (box sums, conductivity sums, k_o S_o partials, in-plane neighbours)
// to the next plane in registers: one __syncthreads and 13 shared loads per node.
constexpr int KT_TY = 8;
constexpr int KT_RING = 8;  // power of two: slot = (plane - zs + 1) & 7

template <int TX>
__global__ void __launch_bounds__(TX * KT_TY, 3) kp_thermal3d_kernel(Ctx cx, int mode, const double* __restrict__ src,
                                                                  double* __restrict__ dst, int ZC) {
  constexpr int T = TX * KT_TY;
  constexpr int DW = TX + 2, DP = 10 * DW;       // d plane tile with halo
  constexpr int EW = TX + 1, EP = 9 * EW;        // element-layer tile
  constexpr int ND = (DP + T - 1) / T, NE = (EP + T - 1) / T;
  const Geo g = cx.g;
  const int nzc = g.N3 / ZC;
  const int load = blockIdx.z / nzc;
  const int zcI = blockIdx.z - load * nzc;
  if (mode == CG && !cx.st[load].active) return;
  extern __shared__ double ksm[];
  double* D = ksm;                      // [KT_RING][DP]
  double* KA = D + KT_RING * DP;        // [4][EP]
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int tx = t % TX, ty = t / TX;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * KT_TY, zs = zcI * ZC;
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const long long plane = (long long)N1 * N2;
  const double* dv = cg_dir(cx, mode, src, load) + (long long)load * g.n;
  const double k0 = cx.mat[0][0], k1 = cx.mat[1][0];

  int goffD[ND], goffE[NE];
#pragma unroll
  for (int m = 0; m < ND; ++m) {
    const int j = t + m * T;
    const int ly = j / DW, lx = j - ly * DW;
    goffD[m] = ((y0 - 1 + ly + N2) & (N2 - 1)) * N1 + ((x0 - 1 + lx + N1) & (N1 - 1));
  }
#pragma unroll
  for (int m = 0; m < NE; ++m) {
    const int j = t + m * T;
    const int ly = j / EW, lx = j - ly * EW;
    goffE[m] = ((y0 - 1 + ly + N2) & (N2 - 1)) * N1 + ((x0 - 1 + lx + N1) & (N1 - 1));
  }
  auto issue_plane = [&](int p) {  // node plane p -> ring slot
    const int zw = (p + N3) & (N3 - 1);
    double* Ds = D + ((p - zs + 1) & (KT_RING - 1)) * DP;
    const double* base = dv + (long long)zw * plane;
#pragma unroll
    for (int m = 0; m < ND; ++m)
      if (t + m * T < DP) cp_async8(Ds + t + m * T, base + goffD[m]);
  };
  unsigned char phv[NE];
  auto fetch_phase = [&](int layer) {
    const int zw = (layer + N3) & (N3 - 1);
    const uint8_t* base = cx.phase + (long long)zw * plane;
#pragma unroll
    for (int m = 0; m < NE; ++m) phv[m] = (t + m * T < EP) ? __ldg(base + goffE[m]) : 0;
  };
  auto store_kappa = [&](int layer) {
    double* Ks = KA + ((layer - zs + 1) & 3) * EP;
#pragma unroll
    for (int m = 0; m < NE; ++m)
      if (t + m * T < EP) Ks[t + m * T] = phv[m] ? k1 : k0;
  };
  // 3x3 neighbourhood of the thread's node column in plane p (local node (tx+1, ty+1))
  double nb[3][3];
  auto read3x3 = [&](int p) {
    const double* Ds = D + ((p - zs + 1) & (KT_RING - 1)) * DP + ty * DW + tx;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) nb[a][b] = Ds[a * DW + b];
  };
  // element box sums Q[oy][ox] of the plane in nb for the 4 elements around the node
  auto box = [&](double Qo[2][2]) {
    const double P00 = nb[0][0] + nb[0][1], P01 = nb[0][1] + nb[0][2];
    const double P10 = nb[1][0] + nb[1][1], P11 = nb[1][1] + nb[1][2];
    const double P20 = nb[2][0] + nb[2][1], P21 = nb[2][1] + nb[2][2];
    Qo[0][0] = P00 + P10;
    Qo[0][1] = P01 + P11;
    Qo[1][0] = P10 + P20;
    Qo[1][1] = P11 + P21;
  };

  // prologue: planes zs-1 .. zs+3 in flight (one commit group each)
#pragma unroll 1
  for (int p = zs - 1; p <= zs + 3; ++p) {
    if (p <= zs + ZC) issue_plane(p);
    cp_commit();
  }
  fetch_phase(zs - 1);
  store_kappa(zs - 1);
  fetch_phase(zs);
  cp_wait<3>();  // planes zs-1, zs landed (this thread's copies)
  __syncthreads();
  double Qk[2][2], Qn[2][2];
  read3x3(zs - 1);
  box(Qk);
  double dzm = nb[1][1];
  read3x3(zs);
  box(Qn);
  double klo[2][2];
  {
    const double* Kl = KA + ty * EW + tx;  // layer zs-1 lives in slot 0
    klo[0][0] = Kl[0];
    klo[0][1] = Kl[1];
    klo[1][0] = Kl[EW];
    klo[1][1] = Kl[EW + 1];
  }
  double KSlo = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) KSlo = fma(klo[a][b], Qk[a][b] + Qn[a][b], KSlo);
  double Klo = (klo[0][0] + klo[0][1]) + (klo[1][0] + klo[1][1]);
  double Kxlo = klo[0][1] + klo[1][1];
  double Kylo = klo[1][0] + klo[1][1];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) Qk[a][b] = Qn[a][b];
  double di = nb[1][1], dxm = nb[1][0], dxp = nb[1][2], dym = nb[0][1], dyp = nb[2][1];

  double part = 0.0;
  const double hc = g.h / 12.0;
  double* outp = dst + (long long)load * g.n + (long long)(y0 + ty) * N1 + (x0 + tx);
#pragma unroll 1
  for (int k = zs; k < zs + ZC; ++k) {
    if (k + 4 <= zs + ZC) issue_plane(k + 4);
    cp_commit();
    cp_wait<3>();      // plane k+1 landed
    store_kappa(k);    // layer k (fetched one iteration ago)
    if (k + 1 < zs + ZC) fetch_phase(k + 1);
    __syncthreads();
    read3x3(k + 1);
    box(Qn);
    const double* Kh = KA + ((k - zs + 1) & 3) * EP + ty * EW + tx;
    const double a00 = Kh[0], a01 = Kh[1], a10 = Kh[EW], a11 = Kh[EW + 1];  // layer k, [oy][ox]
    double KShi = a00 * (Qk[0][0] + Qn[0][0]);
    KShi = fma(a01, Qk[0][1] + Qn[0][1], KShi);
    KShi = fma(a10, Qk[1][0] + Qn[1][0], KShi);
    KShi = fma(a11, Qk[1][1] + Qn[1][1], KShi);
    const double Khi = (a00 + a01) + (a10 + a11);
    const double Kxhi = a01 + a11, Kyhi = a10 + a11;
    const double Ksum = Klo + Khi;
    const double Kxp = Kxlo + Kxhi, Kyp = Kylo + Kyhi;
    const double dzp = nb[1][1];
    double EE = Kxp * dxp;
    EE = fma(Ksum - Kxp, dxm, EE);
    EE = fma(Kyp, dyp, EE);
    EE = fma(Ksum - Kyp, dym, EE);
    EE = fma(Khi, dzp, EE);
    EE = fma(Klo, dzm, EE);
    const double pv = hc * (fma(5.0 * di, Ksum, EE) - (KSlo + KShi));
    outp[(long long)k * plane] = pv;
    part = fma(di, pv, part);
    // carry layer k / plane k+1 into the next step
    KSlo = KShi;
    Klo = Khi;
    Kxlo = Kxhi;
    Kylo = Kyhi;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) Qk[a][b] = Qn[a][b];
    dzm = di;
    di = nb[1][1];
    dxm = nb[1][0];
    dxp = nb[1][2];
    dym = nb[0][1];
    dyp = nb[2][1];
  }
  cp_wait<0>();
  const int nblk = gridDim.x * gridDim.y * nzc;
  const int my = (zcI * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  dp_finish(cx, load, nblk, my, part, red_sh, mode);
}

// Production variant for N1 >= 32: 128 threads own a 32 x 8 node tile, each thread TWO
// vertically adjacent node columns (rows 2ty, 2ty+1).  The two nodes share 6 of their 8 box
// sums and conductivities, so a thread reads a 4x3 block of the next plane (12 loads) and
// 6 conductivities per plane for 2 nodes, and the per-plane bookkeeping (cp.async issue,
// phase fetch, barrier) is amortised over twice the work.
constexpr int KR2_DW = 36, KR2_DPL = 10 * KR2_DW, KR2_PW = 64, KR2_PHS = 9 * KR2_PW;
struct KR2State {   // everything a thread carries from node plane k to k+1 (two node rows)
  double Qk[3][2];                       // box sums of element rows 0..2 (cols 0,1), plane k
  double KSlo[2], Klo[2], Kxlo[2], Kylo[2];  // layer k-1 sums for node 0 / node 1
  double c0, c1, ym, yp, xm0, xp0, xm1, xp1, dzm0, dzm1;  // in-plane values of plane k, centres of k-1
};

template <int TX, int LA>  // LA: planes of cp.async lookahead (< KT_RING)
__global__ void __launch_bounds__(TX * KT_TY / 2, 4) kp_thermal3d_r2_kernel(Ctx cx, int mode,
                                                                          const double* __restrict__ src,
                                                                          double* __restrict__ dst, int ZC,
                                                                          int zc0, int nzl) {
  static_assert(TX == 32, "16-byte staging assumes a 32-wide tile");
  constexpr int T = TX * KT_TY / 2;
  constexpr int DW = KR2_DW;              // staged d row: x0-2 .. x0+33 (16-byte aligned copies)
  constexpr int DPL = KR2_DPL;            // doubles per ring slot (10 rows)
  constexpr int NCH = 10 * (DW / 2);      // 16-byte chunks of d per plane
  constexpr int NDC = (NCH + T - 1) / T;  // per thread
  constexpr int PW = KR2_PW;              // staged phase row: x0-16 .. x0+47 (bytes)
  constexpr int PHS = KR2_PHS;            // phase bytes per ring slot (9 rows)
  constexpr int NPC = PHS / 16;           // 16-byte chunks of phase per plane
  const Geo g = cx.g;
  const int nzc = (g.P3 + ZC - 1) / ZC;
  const int load = blockIdx.z / nzl;                // launch covers z-chunks [zc0, zc0 + nzl)
  const int zcI = zc0 + (blockIdx.z - load * nzl);
  const int dz = g.dirz;  // Dirichlet z: node planes 1..N3-1 stored at index p-1; planes 0, N3 are zero
  if (mode == CG && !cx.st[load].active) return;
  extern __shared__ double ksm[];
  double* D = ksm;  // [KT_RING][10][DW]
  // phase bytes of element layer p-1 travel with node plane p
  unsigned char* PH = reinterpret_cast<unsigned char*>(D + KT_RING * DPL);  // [KT_RING][9][PW]
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int tx = t % TX, ty = t / TX;   // node rows 2ty, 2ty+1 of the tile
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * KT_TY, zs = zcI * ZC + dz;
  const int ze = min(zs + ZC, g.P3 + dz);  // node planes [zs, ze)
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const long long plane = (long long)N1 * N2;
  const double* dv = cg_dir(cx, mode, src, load) + (long long)load * g.n;
  const double k0 = cx.mat[0][0], k1 = cx.mat[1][0];
  // per-thread 16-byte copy assignment (indices past the tile are clamped: harmless duplicates);
  // x pairs start at even x so every chunk stays contiguous across the periodic wrap
  int goffD[NDC];
  unsigned sD[NDC];
#pragma unroll
  for (int m = 0; m < NDC; ++m) {
    const int j = min(t + m * T, NCH - 1);
    const int ly = j / (DW / 2), q = j - ly * (DW / 2);
    goffD[m] = ((y0 - 1 + ly + N2) & (N2 - 1)) * N1 + ((x0 - 2 + 2 * q + N1) & (N1 - 1));
    sD[m] = (unsigned)__cvta_generic_to_shared(D + ly * DW + 2 * q);
  }
  const bool phw = t < NPC;
  const int pj = phw ? t : 0;
  const int prow = pj / (PW / 16), pq = pj - prow * (PW / 16);
  const int poff = ((y0 - 1 + prow + N2) & (N2 - 1)) * N1 + ((x0 - 16 + 16 * pq + N1) & (N1 - 1));
  const unsigned psm = (unsigned)__cvta_generic_to_shared(PH + prow * PW + 16 * pq);
  constexpr unsigned SLOTB = DPL * 8;  // bytes per D ring slot
  auto issue_plane = [&](int p) {  // node plane p of d and phase layer p-1 -> ring slot
    const unsigned slot = (p - zs + 1) & (KT_RING - 1);
    const unsigned so = slot * SLOTB;
    if (dz && (p <= 0 || p >= N3)) {  // fixed (zero) Dirichlet node plane (Fig 4)
#pragma unroll
      for (int m = 0; m < NDC; ++m)
        asm volatile("st.shared.v2.f64 [%0], {0d0000000000000000, 0d0000000000000000};\n" ::"r"(sD[m] + so) : "memory");
    } else {
      const int zw = dz ? p - 1 : ((p + N3) & (N3 - 1));
      const double* base = dv + (long long)zw * plane;
#pragma unroll
      for (int m = 0; m < NDC; ++m)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sD[m] + so), "l"(base + goffD[m]) : "memory");
    }
    if (phw) {
      const uint8_t* pb = cx.phase + (long long)((p - 1 + N3) & (N3 - 1)) * plane + poff;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(psm + slot * PHS), "l"(pb) : "memory");
    }
  };
  double nb[4][3];
  auto read4x3 = [&](int p) {
    const double* Ds = D + ((p - zs + 1) & (KT_RING - 1)) * DPL + 2 * ty * DW + tx + 1;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) nb[a][b] = Ds[a * DW + b];
  };
  auto box = [&](double Qo[3][2]) {
    double P[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      P[a][0] = nb[a][0] + nb[a][1];
      P[a][1] = nb[a][1] + nb[a][2];
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      Qo[e][0] = P[e][0] + P[e + 1][0];
      Qo[e][1] = P[e][1] + P[e + 1][1];
    }
  };
  auto kap6 = [&](int layer, double a[3][2]) {  // layer travels with plane layer+1
    const unsigned char* Pl = PH + ((layer + 1 - zs + 1) & (KT_RING - 1)) * PHS + 2 * ty * PW + tx + 15;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      a[e][0] = Pl[e * PW] ? k1 : k0;
      a[e][1] = Pl[e * PW + 1] ? k1 : k0;
    }
  };
  static_assert(LA >= 2 && LA < KT_RING, "ring slot of plane k+LA must not be read at step k-1");
#pragma unroll 1
  for (int p = zs - 1; p <= zs + LA - 1; ++p) {
    if (p <= ze) issue_plane(p);
    cp_commit();
  }
  cp_wait<LA - 1>();
  __syncthreads();
  KR2State A, B;
  {
    double Qn[3][2], kl[3][2];
    read4x3(zs - 1);
    box(A.Qk);
    A.dzm0 = nb[1][1];
    A.dzm1 = nb[2][1];
    read4x3(zs);
    box(Qn);
    kap6(zs - 1, kl);
    double KS[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) KS[e] = fma(kl[e][0], A.Qk[e][0] + Qn[e][0], kl[e][1] * (A.Qk[e][1] + Qn[e][1]));
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      A.KSlo[m] = KS[m] + KS[m + 1];
      A.Klo[m] = (kl[m][0] + kl[m][1]) + (kl[m + 1][0] + kl[m + 1][1]);
      A.Kxlo[m] = kl[m][1] + kl[m + 1][1];
      A.Kylo[m] = kl[m + 1][0] + kl[m + 1][1];
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      A.Qk[e][0] = Qn[e][0];
      A.Qk[e][1] = Qn[e][1];
    }
    A.c0 = nb[1][1];
    A.c1 = nb[2][1];
    A.ym = nb[0][1];
    A.yp = nb[3][1];
    A.xm0 = nb[1][0];
    A.xp0 = nb[1][2];
    A.xm1 = nb[2][0];
    A.xp1 = nb[2][2];
  }
  double part = 0.0;
  const double hc = g.h * (1.0 / 12.0);
  double* outp = dst + (long long)load * g.n + (long long)(y0 + 2 * ty) * N1 + (x0 + tx);
  // one node plane: reads state `I`, writes the carried state for plane k+1 into `O`
  auto step = [&](int k, const KR2State& I, KR2State& O) {
    if (k + LA <= ze) issue_plane(k + LA);
    cp_commit();
    cp_wait<LA - 1>();
    __syncthreads();
    read4x3(k + 1);
    box(O.Qk);
    double a[3][2];
    kap6(k, a);
    double KS[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) KS[e] = fma(a[e][0], I.Qk[e][0] + O.Qk[e][0], a[e][1] * (I.Qk[e][1] + O.Qk[e][1]));
    const double cz0 = nb[1][1], cz1 = nb[2][1];  // plane k+1 centres
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const double KShi = KS[m] + KS[m + 1];
      const double Khi = (a[m][0] + a[m][1]) + (a[m + 1][0] + a[m + 1][1]);
      const double Kxhi = a[m][1] + a[m + 1][1], Kyhi = a[m + 1][0] + a[m + 1][1];
      const double Ksum = I.Klo[m] + Khi;
      const double Kxp = I.Kxlo[m] + Kxhi, Kyp = I.Kylo[m] + Kyhi;
      const double di = m ? I.c1 : I.c0;
      const double dxp = m ? I.xp1 : I.xp0, dxm = m ? I.xm1 : I.xm0;
      const double dyp = m ? I.yp : I.c1, dym = m ? I.c0 : I.ym;
      const double dzp = m ? cz1 : cz0, dzm = m ? I.dzm1 : I.dzm0;
      double EE = Kxp * dxp;
      EE = fma(Ksum - Kxp, dxm, EE);
      EE = fma(Kyp, dyp, EE);
      EE = fma(Ksum - Kyp, dym, EE);
      EE = fma(Khi, dzp, EE);
      EE = fma(I.Klo[m], dzm, EE);
      double pv = hc * (fma(5.0 * di, Ksum, EE) - (I.KSlo[m] + KShi));
      if (g.dir3 && (x0 + tx == 0 || y0 + 2 * ty + m == 0 || k == 0)) pv = 0.0;  // Dirichlet nodes
      outp[(long long)(k - dz) * plane + m * N1] = pv;
      part = fma(di, pv, part);
      O.KSlo[m] = KShi;
      O.Klo[m] = Khi;
      O.Kxlo[m] = Kxhi;
      O.Kylo[m] = Kyhi;
    }
    O.dzm0 = I.c0;
    O.dzm1 = I.c1;
    O.c0 = cz0;
    O.c1 = cz1;
    O.ym = nb[0][1];
    O.yp = nb[3][1];
    O.xm0 = nb[1][0];
    O.xp0 = nb[1][2];
    O.xm1 = nb[2][0];
    O.xp1 = nb[2][2];
  };
  int k = zs;
#pragma unroll 1
  for (; k + 1 < ze; k += 2) {  // unrolled by two: the carried state ping-pongs A <-> B
    step(k, A, B);
    step(k + 1, B, A);
  }
  if (k < ze) step(k, A, B);
  cp_wait<0>();
  const int nblk = gridDim.x * gridDim.y * nzc;
  const int my = (zcI * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  dp_finish(cx, load, nblk, my, part, red_sh, mode);
}

// Generalisation of the r2 kernel to NR node rows per thread (128 threads, 32 x 4NR node tile):
// the per-plane bookkeeping (ring slot, cp.async issue, barrier, loop) and the box/kappa sums
// shared between vertically adjacent nodes are amortised over NR nodes, so the kernel issues
// fewer instructions per node (it is issue-bound: ncu 65 % issue, 56 % LSU at NR = 2).
template <int NR>
struct KRNState {
  double Qk[NR + 1][2];
  double KSlo[NR], Klo[NR], Kxlo[NR], Kylo[NR];
  double c[NR], xm[NR], xp[NR], dzm[NR];
  double ym, yp;
};

// HALO: slab mode (neighbour planes from Ctx::hlo/hhi); D3: all-Dirichlet output mask.  Both are
// template flags so the common periodic instance carries none of their per-plane logic.
template <int NR, bool HALO, bool D3>
__global__ void __launch_bounds__(128, 2) kp_thermal3d_rn_kernel(Ctx cx, int mode, const double* __restrict__ src,
                                                                double* __restrict__ dst, int ZC, int zc0, int nzl) {
  constexpr int LA = 4;
  constexpr int T = 128, TX = 32, TH = 4 * NR;  // tile: 32 x TH nodes
  constexpr int DW = KR2_DW, DR = TH + 2, DPL = DR * DW;  // d rows y0-1 .. y0+TH
  constexpr int NCH = DR * (DW / 2);
  constexpr int NDC = (NCH + T - 1) / T;
  constexpr int PW = KR2_PW, PR = TH + 1, PHS = PR * PW;  // phase rows y0-1 .. y0+TH-1
  constexpr int NPC = PHS / 16;
  constexpr int NPCT = (NPC + T - 1) / T;
  const Geo g = cx.g;
  const int nzc = (g.P3 + ZC - 1) / ZC;
  // load fastest along grid z: the nrhs CTAs of a tile read the same phase bytes close together
  // in time (L2 hits instead of one HBM read of the phase field per load)
  const int load = blockIdx.z % g.nrhs;
  const int zcI = zc0 + blockIdx.z / g.nrhs;
  const int dz = g.dirz;
  if (mode == CG && !cx.st[load].active) return;
  extern __shared__ double ksm[];
  double* D = ksm;                                                          // [KT_RING][DR][DW]
  unsigned char* PH = reinterpret_cast<unsigned char*>(D + KT_RING * DPL);  // [KT_RING][PR][PW]
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int tx = t % TX, ty = t / TX;  // node rows NR ty .. NR ty + NR - 1
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TH, zs = zcI * ZC + dz + g.zlo;
  const int ze = min(zs + ZC, g.P3 + dz + g.zlo);  // slab mode: global node planes [zlo, zlo + P3)
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const long long plane = (long long)N1 * N2;
  const double* dv = cg_dir(cx, mode, src, load) + (long long)load * g.n;
  const double k0 = cx.mat[0][0], k1 = cx.mat[1][0];
  int goffD[NDC];
  unsigned sD[NDC];
#pragma unroll
  for (int m = 0; m < NDC; ++m) {
    const int j = min(t + m * T, NCH - 1);
    const int ly = j / (DW / 2), q = j - ly * (DW / 2);
    goffD[m] = ((y0 - 1 + ly + N2) & (N2 - 1)) * N1 + ((x0 - 2 + 2 * q + N1) & (N1 - 1));
    sD[m] = (unsigned)__cvta_generic_to_shared(D + ly * DW + 2 * q);
  }
  int poff[NPCT];
  unsigned psm[NPCT];
#pragma unroll
  for (int m = 0; m < NPCT; ++m) {
    const int j = min(t + m * T, NPC - 1);
    const int prow = j / (PW / 16), pq = j - prow * (PW / 16);
    poff[m] = ((y0 - 1 + prow + N2) & (N2 - 1)) * N1 + ((x0 - 16 + 16 * pq + N1) & (N1 - 1));
    psm[m] = (unsigned)__cvta_generic_to_shared(PH + prow * PW + 16 * pq);
  }
  constexpr unsigned SLOTB = DPL * 8;
  auto issue_plane = [&](int p) {
    const unsigned slot = (p - zs + 1) & (KT_RING - 1);
    const unsigned so = slot * SLOTB;
    if (dz && (p <= 0 || p >= N3)) {
#pragma unroll
      for (int m = 0; m < NDC; ++m)
        asm volatile("st.shared.v2.f64 [%0], {0d0000000000000000, 0d0000000000000000};\n" ::"r"(sD[m] + so) : "memory");
    } else {
      const double* base;
      if (HALO)  // slab: neighbours' boundary planes arrive in separate halo buffers
        base = p < g.zlo ? cx.hlo + (long long)load * plane
                         : (p >= g.zlo + g.P3 ? cx.hhi + (long long)load * plane : dv + (long long)(p - g.zlo) * plane);
      else
        base = dv + (long long)(dz ? p - 1 : ((p + N3) & (N3 - 1))) * plane;
#pragma unroll
      for (int m = 0; m < NDC; ++m)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sD[m] + so), "l"(base + goffD[m]) : "memory");
    }
    const uint8_t* pbase = cx.phase + (long long)((p - 1 + N3) & (N3 - 1)) * plane;
#pragma unroll
    for (int m = 0; m < NPCT; ++m)
      if (m * T + t < NPC)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(psm[m] + slot * PHS), "l"(pbase + poff[m]) : "memory");
  };
  double nb[NR + 2][3];
  auto readn = [&](int p) {
    const double* Ds = D + ((p - zs + 1) & (KT_RING - 1)) * DPL + NR * ty * DW + tx + 1;
#pragma unroll
    for (int a = 0; a < NR + 2; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) nb[a][b] = Ds[a * DW + b];
  };
  auto box = [&](double Qo[NR + 1][2]) {
    double P[NR + 2][2];
#pragma unroll
    for (int a = 0; a < NR + 2; ++a) {
      P[a][0] = nb[a][0] + nb[a][1];
      P[a][1] = nb[a][1] + nb[a][2];
    }
#pragma unroll
    for (int e = 0; e < NR + 1; ++e) {
      Qo[e][0] = P[e][0] + P[e + 1][0];
      Qo[e][1] = P[e][1] + P[e + 1][1];
    }
  };
  auto kap = [&](int layer, double a[NR + 1][2]) {
    const unsigned char* Pl = PH + ((layer + 1 - zs + 1) & (KT_RING - 1)) * PHS + NR * ty * PW + tx + 15;
#pragma unroll
    for (int e = 0; e < NR + 1; ++e) {
      a[e][0] = Pl[e * PW] ? k1 : k0;
      a[e][1] = Pl[e * PW + 1] ? k1 : k0;
    }
  };
#pragma unroll 1
  for (int p = zs - 1; p <= zs + LA - 1; ++p) {
    if (p <= ze) issue_plane(p);
    cp_commit();
  }
  cp_wait<LA - 1>();
  __syncthreads();
  KRNState<NR> A, B;
  {
    double Qn[NR + 1][2], kl[NR + 1][2];
    readn(zs - 1);
    box(A.Qk);
#pragma unroll
    for (int m = 0; m < NR; ++m) A.dzm[m] = nb[m + 1][1];
    readn(zs);
    box(Qn);
    kap(zs - 1, kl);
    double KS[NR + 1];
#pragma unroll
    for (int e = 0; e < NR + 1; ++e) KS[e] = fma(kl[e][0], A.Qk[e][0] + Qn[e][0], kl[e][1] * (A.Qk[e][1] + Qn[e][1]));
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      A.KSlo[m] = KS[m] + KS[m + 1];
      A.Klo[m] = (kl[m][0] + kl[m][1]) + (kl[m + 1][0] + kl[m + 1][1]);
      A.Kxlo[m] = kl[m][1] + kl[m + 1][1];
      A.Kylo[m] = kl[m + 1][0] + kl[m + 1][1];
      A.c[m] = nb[m + 1][1];
      A.xm[m] = nb[m + 1][0];
      A.xp[m] = nb[m + 1][2];
    }
#pragma unroll
    for (int e = 0; e < NR + 1; ++e) {
      A.Qk[e][0] = Qn[e][0];
      A.Qk[e][1] = Qn[e][1];
    }
    A.ym = nb[0][1];
    A.yp = nb[NR + 1][1];
  }
  double part = 0.0;
  const double hc = g.h * (1.0 / 12.0);
  double* outp = dst + (long long)load * g.n + (long long)(y0 + NR * ty) * N1 + (x0 + tx);
  // Dirichlet-node mask bits of this thread's NR nodes (all-Dirichlet storage), loop invariant
  unsigned fixed_xy = 0;
  if (D3)
#pragma unroll
    for (int m = 0; m < NR; ++m)
      if (x0 + tx == 0 || y0 + NR * ty + m == 0) fixed_xy |= 1u << m;
  auto step = [&](int k, const KRNState<NR>& I, KRNState<NR>& O) {
    if (k + LA <= ze) issue_plane(k + LA);
    cp_commit();
    cp_wait<LA - 1>();
    __syncthreads();
    readn(k + 1);
    box(O.Qk);
    double a[NR + 1][2];
    kap(k, a);
    double KS[NR + 1];
#pragma unroll
    for (int e = 0; e < NR + 1; ++e) KS[e] = fma(a[e][0], I.Qk[e][0] + O.Qk[e][0], a[e][1] * (I.Qk[e][1] + O.Qk[e][1]));
    double* orow = outp + (long long)(k - dz - g.zlo) * plane;
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      const double KShi = KS[m] + KS[m + 1];
      const double Khi = (a[m][0] + a[m][1]) + (a[m + 1][0] + a[m + 1][1]);
      const double Kxhi = a[m][1] + a[m + 1][1], Kyhi = a[m + 1][0] + a[m + 1][1];
      const double Ksum = I.Klo[m] + Khi;
      const double Kxp = I.Kxlo[m] + Kxhi, Kyp = I.Kylo[m] + Kyhi;
      const double di = I.c[m];
      const double dyp = m + 1 < NR ? I.c[m + 1] : I.yp, dym = m > 0 ? I.c[m - 1] : I.ym;
      const double dzp = nb[m + 1][1];  // plane k+1 centre
      double EE = Kxp * I.xp[m];
      EE = fma(Ksum - Kxp, I.xm[m], EE);
      EE = fma(Kyp, dyp, EE);
      EE = fma(Ksum - Kyp, dym, EE);
      EE = fma(Khi, dzp, EE);
      EE = fma(I.Klo[m], I.dzm[m], EE);
      double pv = hc * (fma(5.0 * di, Ksum, EE) - (I.KSlo[m] + KShi));
      if (D3 && (((fixed_xy >> m) & 1u) || k == 0)) pv = 0.0;  // Dirichlet nodes
      if (HALO && g.zpad && k == 0) pv = 0.0;                    // slab Dirichlet-z face (padded)
      orow[m * N1] = pv;
      part = fma(di, pv, part);
      O.KSlo[m] = KShi;
      O.Klo[m] = Khi;
      O.Kxlo[m] = Kxhi;
      O.Kylo[m] = Kyhi;
    }
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      O.dzm[m] = I.c[m];
      O.c[m] = nb[m + 1][1];
      O.xm[m] = nb[m + 1][0];
      O.xp[m] = nb[m + 1][2];
    }
    O.ym = nb[0][1];
    O.yp = nb[NR + 1][1];
  };
  int k = zs;
#pragma unroll 1
  for (; k + 1 < ze; k += 2) {
    step(k, A, B);
    step(k + 1, B, A);
  }
  if (k < ze) step(k, A, B);
  cp_wait<0>();
  const int nblk = gridDim.x * gridDim.y * nzc;
  const int my = (zcI * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  dp_finish(cx, load, nblk, my, part, red_sh, mode);
}

// rows per thread of the production thermal 3D K kernel (4; 2 when N2 < 16)
static int k_nr(const Geo& g) { return g.N2 >= 16 ? 4 : 2; }


// Thermal 2D: element row (App. A1: {2/3, -1/6, -1/3}) ->
//   p_i = 1/6 [ 6 d_i sum_o k_o + sum_{4 axis nbrs} d_j (k of the 2 octants on edge ij) - 2 sum_o k_o S_o ].
__global__ void __launch_bounds__(256) kp_thermal2d_kernel(Ctx cx, int mode, const double* __restrict__ src,
                                                           double* __restrict__ dst) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (mode == CG && !cx.st[load].active) return;
  __shared__ double red_sh[32];
  const int N1 = g.N1, N2 = g.N2;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double part = 0.0;
  if (i < g.n) {
    const int x = (int)(i % N1), y = (int)(i / N1);
    const double* dv = cg_dir(cx, mode, src, load) + (long long)load * g.n;
    const int xm = (x - 1 + N1) & (N1 - 1), xp = (x + 1) & (N1 - 1), ym = (y - 1 + N2) & (N2 - 1), yp = (y + 1) & (N2 - 1);
    auto D = [&](int xx, int yy) { return __ldg(dv + (long long)yy * N1 + xx); };
    auto KAP = [&](int xx, int yy) { return __ldg(cx.phase + (long long)yy * N1 + xx) ? cx.mat[1][0] : cx.mat[0][0]; };
    const double a00 = KAP(xm, ym), a01 = KAP(x, ym), a10 = KAP(xm, y), a11 = KAP(x, y);  // [oy][ox]
    const double dmm = D(xm, ym), d0m = D(x, ym), dpm = D(xp, ym);
    const double dm0 = D(xm, y), d00 = D(x, y), dp0 = D(xp, y);
    const double dmp = D(xm, yp), d0p = D(x, yp), dpp = D(xp, yp);
    const double S00 = (dmm + d0m) + (dm0 + d00), S01 = (d0m + dpm) + (d00 + dp0);
    const double S10 = (dm0 + d00) + (dmp + d0p), S11 = (d00 + dp0) + (d0p + dpp);
    const double Ksum = (a00 + a01) + (a10 + a11);
    const double KS = fma(a00, S00, fma(a01, S01, fma(a10, S10, a11 * S11)));
    double EE = (a01 + a11) * dp0;
    EE = fma(a00 + a10, dm0, EE);
    EE = fma(a10 + a11, d0p, EE);
    EE = fma(a00 + a01, d0m, EE);
    double pv = (fma(6.0 * d00, Ksum, EE) - 2.0 * KS) * (1.0 / 6.0);
    if (((g.dmask & 1) && x == 0) || ((g.dmask & 2) && y == 0)) pv = 0.0;  // Dirichlet nodes (padded storage)
    dst[(long long)load * g.n + i] = pv;
    part = d00 * pv;
  }
  dp_finish(cx, load, gridDim.x, blockIdx.x, part, red_sh, mode);
}


__global__ void __launch_bounds__(256) kp_elastic2d_kernel(Ctx cx, int mode, const double* __restrict__ src,
                                                           double* __restrict__ dst) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (mode == CG && !cx.st[load].active) return;
  __shared__ double red_sh[32];
  const int N1 = g.N1, N2 = g.N2;
  const long long n = g.n;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double part = 0.0;
  if (i < n) {
    const int x = (int)(i % N1), y = (int)(i / N1);
    const double* dv = cg_dir(cx, mode, src, load) + (long long)load * 2 * n;
    double acc[2] = {0.0, 0.0};
    for (int o = 0; o < 4; ++o) {
      const int ox = o & 1, oy = o >> 1;
      const int a = (1 - ox) + 2 * (1 - oy);
      const int ex = (x - 1 + ox + N1) & (N1 - 1), ey = (y - 1 + oy + N2) & (N2 - 1);
      const int ph = __ldg(cx.phase + (long long)ey * N1 + ex) ? 1 : 0;
      for (int b = 0; b < 4; ++b) {
        const int bx = b & 1, by = b >> 1;
        const int nx = (ex + bx) & (N1 - 1), ny = (ey + by) & (N2 - 1);
        const double u0 = __ldg(dv + (long long)ny * N1 + nx), u1 = __ldg(dv + n + (long long)ny * N1 + nx);
        for (int al = 0; al < 2; ++al) {
          const double* row = cx.kel + ph * 64 + (2 * a + al) * 8 + 2 * b;
          acc[al] = fma(__ldg(row), u0, fma(__ldg(row + 1), u1, acc[al]));
        }
      }
    }
    if (((g.dmask & 1) && x == 0) || ((g.dmask & 2) && y == 0)) acc[0] = acc[1] = 0.0;  // Dirichlet nodes
    for (int al = 0; al < 2; ++al) {
      dst[(long long)load * 2 * n + al * n + i] = acc[al];
      part = fma(__ldg(dv + al * n + i), acc[al], part);
    }
  }
  dp_finish(cx, load, gridDim.x, blockIdx.x, part, red_sh, mode);
}

// ============================================================================== RHS (Eq 76 / 81)
// f_(i,alpha) = -(h^(d-1)/2^(d-1)) sum_o sum_j s_j(o) sigma^o_(alpha j),  s_j(o) = +1 if o_j = 0 else -1,
// sigma^o = kappa_o g_bar (thermal, alpha = 0) or lambda_o tr(eps) I + 2 mu_o eps (elastic).

// octant phases of node i (stored index), shift-based decode (N1, N2 powers of two)
__device__ __forceinline__ unsigned node_octants(const Ctx& cx, long long i, int& z) {
  const Geo& g = cx.g;
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const int s1 = __ffs(N1) - 1, s2 = __ffs(N2) - 1;
  const int x = (int)(i & (N1 - 1));
  const int y = (int)((i >> s1) & (N2 - 1));
  z = (int)(i >> (s1 + s2)) + g.dirz + g.zlo;  // Dirichlet z: stored planes are nodes 1..N3-1; slab offset
  unsigned bits = 0;
  const int no = 1 << g.dim;
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    if (o >= no) break;
    const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
    const int ex = (x - 1 + ox) & (N1 - 1), ey = (y - 1 + oy) & (N2 - 1);
    const int ez = g.dim == 3 ? (z - 1 + oz + N3) % N3 : 0;
    bits |= (__ldg(cx.phase + ((long long)ez * N2 + ey) * N1 + ex) ? 1u : 0u) << o;
  }
  return bits;
}

// Since sum_o s_j(o) = 0, only the phase contrast survives: with the per-node integers
//   n_j = sum_o s_j(o) [phase_o = 1]   (in [-2^(d-1), 2^(d-1)]),
// f_(i,alpha) = sum_j C[l][alpha][j] n_j with C = -(h^(d-1)/2^(d-1)) * { (k1 - k0) g_bar_j  (thermal);
// (lam1 - lam0) tr(eps) delta_(alpha j) + 2 (mu1 - mu0) eps_(alpha j)  (elastic) }.
__device__ void rhs_coef(const Ctx& cx, const LoadParams& lp, double* C /* [nrhs][c][3] */) {
  const Geo& g = cx.g;
  const int d = g.dim, c = g.c, nl = g.nrhs;
  const double scale = (d == 3 ? g.h * g.h / 4.0 : g.h / 2.0);
  const double rt2 = 0.70710678118654752440;
  for (int idx = threadIdx.x; idx < nl * c * 3; idx += blockDim.x) {
    const int j = idx % 3, al = (idx / 3) % c, l = idx / (3 * c);
    double v = 0.0;
    if (j < d) {
      if (c == 1) {
        v = (cx.mat[1][0] - cx.mat[0][0]) * lp.v[l][j];
      } else {
        double e[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        if (d == 3) {
          e[0][0] = lp.v[l][0]; e[1][1] = lp.v[l][1]; e[2][2] = lp.v[l][2];
          e[0][1] = e[1][0] = lp.v[l][3] * rt2;
          e[0][2] = e[2][0] = lp.v[l][4] * rt2;
          e[1][2] = e[2][1] = lp.v[l][5] * rt2;
        } else {
          e[0][0] = lp.v[l][0]; e[1][1] = lp.v[l][1];
          e[0][1] = e[1][0] = lp.v[l][2] * rt2;
        }
        const double tr = e[0][0] + e[1][1] + e[2][2];
        v = (al == j ? (cx.mat[1][0] - cx.mat[0][0]) * tr : 0.0) + 2.0 * (cx.mat[1][1] - cx.mat[0][1]) * e[al][j];
      }
    }
    C[idx] = -scale * v;
  }
  __syncthreads();
}

// Warp variant for 3D grids with N1 % 32 == 0: the 32 lanes hold 32 consecutive x of one row,
// so every lane loads only the 4 voxels (x, y-1..y, z-1..z) and takes the x-1 voxels from its
// left neighbour (lane 0 loads them itself).  All 32 lanes must be active.
__device__ __forceinline__ unsigned node_octants_warp(const Ctx& cx, long long i, int& z) {
  const Geo& g = cx.g;
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const int s1 = __ffs(N1) - 1, s2 = __ffs(N2) - 1;
  const int lane = threadIdx.x & 31;
  const int x = (int)(i & (N1 - 1));
  const int y = (int)((i >> s1) & (N2 - 1));
  z = (int)(i >> (s1 + s2)) + g.dirz + g.zlo;
  const int ym = (y - 1) & (N2 - 1);
  const int zm = g.dirz ? z - 1 : ((z - 1) & (N3 - 1));
  const int zp = z;  // voxel layer z (node planes 0..N3-1 periodic, 1..N3-1 Dirichlet: no wrap)
  const uint8_t* p00 = cx.phase + ((long long)zm * N2 + ym) * N1;  // [oz=0][oy=0]
  const uint8_t* p01 = cx.phase + ((long long)zm * N2 + y) * N1;   // [oz=0][oy=1]
  const uint8_t* p10 = cx.phase + ((long long)zp * N2 + ym) * N1;  // [oz=1][oy=0]
  const uint8_t* p11 = cx.phase + ((long long)zp * N2 + y) * N1;   // [oz=1][oy=1]
  const unsigned b00 = __ldg(p00 + x) != 0, b01 = __ldg(p01 + x) != 0, b10 = __ldg(p10 + x) != 0,
                 b11 = __ldg(p11 + x) != 0;
  // octant o = ox + 2 oy + 4 oz; ox = 1 is voxel x, ox = 0 voxel x - 1
  unsigned hi = (b00 << 1) | (b01 << 3) | (b10 << 5) | (b11 << 7);
  unsigned lo = __shfl_up_sync(0xffffffffu, hi, 1) >> 1;
  if (lane == 0) {
    const int xm = (x - 1) & (N1 - 1);
    lo = (__ldg(p00 + xm) != 0) | ((__ldg(p01 + xm) != 0) << 2) | ((__ldg(p10 + xm) != 0) << 4) |
         ((__ldg(p11 + xm) != 0) << 6);
  }
  return hi | lo;
}

__device__ __forceinline__ void octant_counts(unsigned bits, int d, int n[3]) {
  n[0] = n[1] = n[2] = 0;
#pragma unroll
  for (int o = 0; o < 8; ++o) {  // bits of absent octants (2D: o >= 4) are zero
    const int b = (bits >> o) & 1;
    n[0] += (o & 1) ? -b : b;
    n[1] += (o & 2) ? -b : b;
    n[2] += (o & 4) ? -b : b;
  }
  if (d == 2) n[2] = 0;
}

__global__ void __launch_bounds__(256) rhs_kernel(Ctx cx, LoadParams lp, double* __restrict__ f) {
  __shared__ double C[kMaxRhs * 3 * 3];
  const Geo g = cx.g;
  rhs_coef(cx, lp, C);
  const int nl = g.nrhs, c = g.c;
  const bool warp_ok = g.dim == 3 && (g.N1 & 31) == 0;  // block-uniform
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (long long)gridDim.x * blockDim.x) {
    int z, n[3];
    octant_counts(warp_ok ? node_octants_warp(cx, i, z) : node_octants(cx, i, z), g.dim, n);
    const double n0 = n[0], n1 = n[1], n2 = n[2];
    const bool fixed = ((g.dmask & 1) && (i & (g.N1 - 1)) == 0) || ((g.dmask & 2) && ((i / g.N1) & (g.N2 - 1)) == 0) ||
                       ((g.dmask & 4) && z == 0);  // Dirichlet node of the padded storage
    for (int l = 0; l < nl; ++l)
      for (int al = 0; al < c; ++al) {
        const double* Cr = C + (l * c + al) * 3;
        f[((long long)l * c + al) * g.n + i] = fixed ? 0.0 : fma(Cr[0], n0, fma(Cr[1], n1, Cr[2] * n2));
      }
  }
}

// ============================================================================== finalize / means
__global__ void finalize_kernel(Ctx cx) {
  const Geo g = cx.g;
  const int load = blockIdx.y;
  const LoadState* st = cx.st + load;
  const long long cnt = (long long)g.c * g.n;
  double* u = cx.u + (long long)load * cnt;
  const double a = st->alpha;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x, stp = (long long)gridDim.x * blockDim.x;
  if (cx.d2) {  // paired u updates: the terms u_done .. iters-1 (one or two) are still owed
    const int I = st->iters, owed = I - st->u_done;
    if (I < 1 || owed <= 0) return;
    auto dir = [&](int j) { return ((j & 1) ? cx.d2 : cx.d) + (long long)load * cnt; };
    const double* dl = dir(I - 1);
    if (owed >= 2) {
      const double* dp = dir(I - 2);
      const double a2 = st->alpha_prev;
      for (long long i = i0; i < cnt; i += stp) u[i] = fma(a, dl[i], fma(a2, dp[i], u[i]));
    } else {
      for (long long i = i0; i < cnt; i += stp) u[i] = fma(a, dl[i], u[i]);
    }
    return;
  }
  if (!st->pending_u || st->iters < 1) return;
  const double* d = cx.d + (long long)load * cnt;
  for (long long i = i0; i < cnt; i += stp) u[i] = fma(a, d[i], u[i]);
}

// per (load, comp) partial sums over fixed chunks, then a fixed-order combine + subtract
__global__ void mean_partial_kernel(const double* __restrict__ u, long long n, double* partials, int nblk) {
  __shared__ double sh[32];
  const int lc = blockIdx.y;
  const double* v = u + (long long)lc * n;
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)nblk * blockDim.x)
    acc += v[i];
  const double b = block_reduce<false>(acc, sh);
  if (threadIdx.x == 0) partials[(long long)lc * nblk + blockIdx.x] = b;
}
__global__ void mean_combine_kernel(const double* partials, int nblk, long long n, double* means) {
  __shared__ double sh[32];
  const int lc = blockIdx.x;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) acc += partials[(long long)lc * nblk + i];
  const double b = block_reduce<false>(acc, sh);
  if (threadIdx.x == 0) means[lc] = b / (double)n;
}
__global__ void mean_subtract_kernel(const double* __restrict__ src, double* __restrict__ dst, long long n,
                                     const double* means) {
  const int lc = blockIdx.y;
  const double m = means[lc];
  const double* v = src + (long long)lc * n;
  double* o = dst + (long long)lc * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    o[i] = v[i] - m;
}

// ============================================================================== effective property
// acc[i][j] = f^(i) . u^(j) (f recomputed per node, never stored); plus the count of phase-1
// voxels for <C>.
constexpr int EFF_T = 256;
// Same quantity through the octant counts: f^(li) . u^(lj) = sum_(alpha, j) C[li][alpha][j] T[lj][alpha][j],
// T[lj][alpha][j] = sum_nodes n_j u^(lj)_alpha accumulated per thread and contracted at the end.
template <int NL, int CC>
__global__ void __launch_bounds__(EFF_T) effective_n_kernel(Ctx cx, LoadParams lp, const double* __restrict__ u,
                                                            double* partials) {
  __shared__ double C[kMaxRhs * 3 * 3];
  __shared__ double sh[32];
  const Geo g = cx.g;
  rhs_coef(cx, lp, C);
  double T[NL][CC][3];
#pragma unroll
  for (int l = 0; l < NL; ++l)
#pragma unroll
    for (int a = 0; a < CC; ++a) T[l][a][0] = T[l][a][1] = T[l][a][2] = 0.0;
  double cnt = 0.0;
  const int no = 1 << g.dim;
  const bool warp_ok = g.dim == 3 && (g.N1 & 31) == 0;  // block-uniform
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (long long)gridDim.x * blockDim.x) {
    int z, n[3];
    const unsigned bits = warp_ok ? node_octants_warp(cx, i, z) : node_octants(cx, i, z);
    cnt += (bits >> (no - 1)) & 1;  // voxel i is octant (1,1,1) of node i: each voxel once
    if (g.dirz && z == 1) cnt += (bits >> 3) & 1;  // Dirichlet z: voxel layer 0
    octant_counts(bits, g.dim, n);
    const double n0 = n[0], n1 = n[1], n2 = n[2];
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
      for (int a = 0; a < CC; ++a) {
        const double uv = u[((long long)l * CC + a) * g.n + i];
        T[l][a][0] = fma(n0, uv, T[l][a][0]);
        T[l][a][1] = fma(n1, uv, T[l][a][1]);
        T[l][a][2] = fma(n2, uv, T[l][a][2]);
      }
  }
#pragma unroll
  for (int li = 0; li < NL; ++li)
#pragma unroll
    for (int lj = 0; lj < NL; ++lj) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < CC; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) acc = fma(C[(li * CC + a) * 3 + j], T[lj][a][j], acc);
      const double b = block_reduce<false>(acc, sh);
      if (threadIdx.x == 0) partials[(long long)(li * NL + lj) * gridDim.x + blockIdx.x] = b;
      __syncthreads();
    }
  const double b = block_reduce<false>(cnt, sh);
  if (threadIdx.x == 0) partials[(long long)(NL * NL) * gridDim.x + blockIdx.x] = b;
}

__global__ void combine_rows_kernel(const double* partials, int nblk, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) acc += partials[(long long)blockIdx.x * nblk + i];
  const double b = block_reduce<false>(acc, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = b;
}

// ============================================================================== symbol (a0)
// G_hat(k)/n on the half spectrum, layout [C][H1][N3][N2].
// Reference symbol (closed form of the Q1 stencil's DFT, App./SURVEY A3 — the oracle probes
// it instead):  S_ii = (2/h)(1-cos t_i) prod_{j!=i} (h/3)(2+cos t_j);
//               S_ij = sin t_i sin t_j prod_{l!=i,j} (h/3)(2+cos t_l).
// thermal A = kappa_r tr S ; elastic A = (lam_r + mu_r) S + mu_r tr(S) I  (Eq 36 symbol).
// Perturbation: c=1 rho = 1-amp+2 amp u01(seed,2,canon(k));
//   c=3 G = Phi + amp tr(Phi)/3 psi(theta), theta_t = u01(seed,2,8 canon(k)+t) (Eq B5);
//   c=2 analogous with Eq 45.  canon(k) = min(flat(k), flat(-k)).  G(0) = 0.
// cos, sin and 1 - cos of theta = 2 pi k / N; 1 - cos is evaluated as 2 sin^2(theta / 2) (no
// cancellation at low frequency, where the symbol ~ theta^2: relative accuracy ~eps on every bin)
__device__ __forceinline__ void axis_trig(int k, int N, double& cs, double& sn, double& omc) {
  const int ks = (2 * k <= N) ? k : k - N;  // signed frequency: cos even, sin odd -> G(-k)=G(k) bitwise
  const int ka = ks < 0 ? -ks : ks;
  double s, c;
  sincospi(2.0 * (double)ka / (double)N, &s, &c);
  cs = c;
  sn = ks < 0 ? -s : s;
  const double sh = sinpi((double)ka / (double)N);
  omc = 2.0 * sh * sh;
}

__global__ void build_symbol_kernel(Ctx cx, double* gtab, double ref0, double ref1, unsigned long long seed, double amp) {
  const Geo g = cx.g;
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nspec) return;
  // N2l: stored k_y extent of this table (a y-chunk in slab mode); N2: the grid's N2 (frequencies)
  const int N1 = g.N1, N2l = g.N2, N2 = g.Ny ? g.Ny : g.N2, N3 = g.N3, d = g.dim;
  int kx, ky, kz;
  if (!g.dirz) {  // 5-pass layout [kx][kz][ky]: powers of two, shifts only
    const int s2 = __ffs(N2l) - 1, s3 = __ffs(N3) - 1;
    ky = (int)(b & (N2l - 1)) + g.ky0;  // y-chunk pencil (slab mode): global k_y
    kz = (int)((b >> s2) & (N3 - 1));
    kx = (int)(b >> (s2 + s3));
  } else {         // mixed layout [kx][sine plane][ky]
    ky = (int)(b % N2l);
    kz = (int)((b / N2l) % g.P3);
    kx = (int)(b / ((long long)N2l * g.P3));
  }
  double cs[3], sn[3], omc[3];
  axis_trig(kx, N1, cs[0], sn[0], omc[0]);
  axis_trig(ky, N2, cs[1], sn[1], omc[1]);
  double inv_n;
  unsigned long long flat, flatm;
  bool zero;
  if (g.dirz || g.zpad) {
    // mixed BC: sine mode m along z (m = kz + 1 on the N3-1 stored sine planes; the
    // slab pencil's padded layout keeps mode m at index kz = m, index 0 held at 0), theta_z = pi m / N3;
    // the odd x-z / y-z couplings leave the diagonal block (S_xz = S_yz = 0); sine modes are
    // self-conjugate, the perturbation is drawn at the sine-plane index p = m - 1.
    const int m = g.zpad ? kz : kz + 1;
    const unsigned long long pz = (unsigned long long)(m > 0 ? m - 1 : 0);
    double sz, cz;
    sincospi((double)m / (double)N3, &sz, &cz);
    cs[2] = cz;
    sn[2] = 0.0;
    const double shz = sinpi((double)m / (2.0 * N3));
    omc[2] = 2.0 * shz * shz;
    inv_n = 2.0 / ((double)N1 * N2 * N3);  // F_x F_y unnormalised (N1 N2) x sine sums (N3/2)
    flat = (pz * N2 + ky) * N1 + kx;
    flatm = (pz * N2 + (unsigned long long)((N2 - ky) % N2)) * N1 + (unsigned long long)((N1 - kx) % N1);
    zero = m == 0;
  } else {
    axis_trig(kz, N3, cs[2], sn[2], omc[2]);
    inv_n = 1.0 / ((double)N1 * N2 * N3);  // = 1/n (N2: the whole grid, also for a y-chunk pencil)
    flat = ((unsigned long long)kz * N2 + ky) * N1 + kx;
    flatm = ((unsigned long long)((N3 - kz) & (N3 - 1)) * N2 + (unsigned long long)((N2 - ky) & (N2 - 1))) * N1 +
            (unsigned long long)((N1 - kx) & (N1 - 1));
    zero = (kx == 0 && ky == 0 && kz == 0);
  }
  const double h = g.h;
  const long long ns = g.nspec;
  const unsigned long long canon = flat < flatm ? flat : flatm;
  if (g.c == 1 && d == 3) {  // thermal 3D in scalars (same operation order as the general path)
    const double m0 = (h / 3.0) * (2.0 + cs[0]), m1 = (h / 3.0) * (2.0 + cs[1]), m2 = (h / 3.0) * (2.0 + cs[2]);
    const double S00 = (2.0 / h) * omc[0] * m1 * m2;
    const double S11 = (2.0 / h) * omc[1] * m0 * m2;
    const double S22 = (2.0 / h) * omc[2] * m0 * m1;
    const double a = (((0.0 + S00) + S11) + S22) * ref0;
    double gv = 0.0;
    if (!zero) {
      const double rho = seed ? (1.0 - amp + 2.0 * amp * u01(seed, 2, canon)) : 1.0;
      gv = rho / a * inv_n;
    }
    gtab[b] = gv;
    return;
  }
  double mass[3], S[3][3];
  for (int i = 0; i < d; ++i) mass[i] = (h / 3.0) * (2.0 + cs[i]);
  for (int i = 0; i < d; ++i) {
    double v = (2.0 / h) * omc[i];
    for (int j = 0; j < d; ++j)
      if (j != i) v *= mass[j];
    S[i][i] = v;
    for (int j = 0; j < d; ++j) {
      if (j == i) continue;
      double w = sn[i] * sn[j];
      for (int l = 0; l < d; ++l)
        if (l != i && l != j) w *= mass[l];
      S[i][j] = w;
    }
  }
  if (g.c == 1) {
    double a = 0.0;
    for (int i = 0; i < d; ++i) a += S[i][i];
    a *= ref0;
    double gv = 0.0;
    if (!zero) {
      const double rho = seed ? (1.0 - amp + 2.0 * amp * u01(seed, 2, canon)) : 1.0;
      gv = rho / a * inv_n;
    }
    gtab[b] = gv;
    return;
  }
  const double lr = ref0, mr = ref1;
  double tr = 0.0;
  for (int i = 0; i < d; ++i) tr += S[i][i];
  double A[3][3];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) A[i][j] = (lr + mr) * S[i][j] + (i == j ? mr * tr : 0.0);
  double P[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  if (!zero) {
    if (d == 3) {
      // symmetric A: inverse from cofactors (A is symmetric by construction)
      const double i00 = A[1][1] * A[2][2] - A[1][2] * A[1][2];
      const double i01 = A[0][2] * A[1][2] - A[0][1] * A[2][2];
      const double i02 = A[0][1] * A[1][2] - A[0][2] * A[1][1];
      const double i11 = A[0][0] * A[2][2] - A[0][2] * A[0][2];
      const double i12 = A[0][2] * A[0][1] - A[0][0] * A[1][2];
      const double i22 = A[0][0] * A[1][1] - A[0][1] * A[0][1];
      const double id = 1.0 / (A[0][0] * i00 + A[0][1] * i01 + A[0][2] * i02);
      P[0][0] = i00 * id;
      P[1][1] = i11 * id;
      P[2][2] = i22 * id;
      P[0][1] = P[1][0] = i01 * id;
      P[0][2] = P[2][0] = i02 * id;
      P[1][2] = P[2][1] = i12 * id;
      if (seed) {
        double th[6];
        for (int tt = 0; tt < 6; ++tt) th[tt] = u01(seed, 2, 8ULL * canon + tt);
        th[0] = 0.5 + 0.5 * th[0];
        th[1] = 0.5 + 0.5 * th[1];
        th[3] = 0.5 + 0.5 * th[3];
        th[2] -= 0.5;
        th[4] -= 0.5;
        th[5] -= 0.5;
        const double t1 = th[0], t2 = th[1], t3 = th[2], t4 = th[3], t5 = th[4], t6 = th[5];
        const double s = amp * (P[0][0] + P[1][1] + P[2][2]) / 3.0;
        const double psi[3][3] = {{t1 * t1, t1 * t3, t1 * t6},
                                  {t1 * t3, t2 * t2 + t3 * t3, t2 * t5 + t3 * t6},
                                  {t1 * t6, t2 * t5 + t3 * t6, t4 * t4 + t5 * t5 + t6 * t6}};
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) P[i][j] += s * psi[i][j];
      }
    } else {
      const double det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
      P[0][0] = A[1][1] / det;
      P[1][1] = A[0][0] / det;
      P[0][1] = P[1][0] = -0.5 * (A[0][1] + A[1][0]) / det;
      if (seed) {
        double t1 = 0.5 + 0.5 * u01(seed, 2, 8ULL * canon + 0);
        double t2 = 0.5 + 0.5 * u01(seed, 2, 8ULL * canon + 1);
        double t3 = u01(seed, 2, 8ULL * canon + 2) - 0.5;
        const double s = amp * (P[0][0] + P[1][1]) / 2.0;
        P[0][0] += s * t1 * t1;
        P[0][1] += s * t1 * t3;
        P[1][0] += s * t1 * t3;
        P[1][1] += s * (t2 * t2 + t3 * t3);
      }
    }
  }
  if (g.c == 3) {
    gtab[0 * ns + b] = P[0][0] * inv_n;
    gtab[1 * ns + b] = P[1][1] * inv_n;
    gtab[2 * ns + b] = P[0][1] * inv_n;
    gtab[3 * ns + b] = P[2][2] * inv_n;
    gtab[4 * ns + b] = P[1][2] * inv_n;
    gtab[5 * ns + b] = P[0][2] * inv_n;
  } else {
    gtab[0 * ns + b] = P[0][0] * inv_n;
    gtab[1 * ns + b] = P[1][1] * inv_n;
    gtab[2 * ns + b] = P[0][1] * inv_n;
  }
}

// Eq 55: min / max block eigenvalue of n*G_hat(k) over k != 0 (2x2 / 3x3 closed forms).
__device__ void eig_sym3(double a, double b, double c, double d, double e, double f, double& lmin, double& lmax) {
  // matrix [[a,d,f],[d,b,e],[f,e,c]]
  const double p1 = d * d + e * e + f * f;
  const double q = (a + b + c) / 3.0;
  const double p2 = (a - q) * (a - q) + (b - q) * (b - q) + (c - q) * (c - q) + 2.0 * p1;
  const double p = sqrt(p2 / 6.0);
  if (p == 0.0) {
    lmin = lmax = q;
    return;
  }
  const double ip = 1.0 / p;
  const double B00 = (a - q) * ip, B11 = (b - q) * ip, B22 = (c - q) * ip, B01 = d * ip, B12 = e * ip, B02 = f * ip;
  double r = 0.5 * (B00 * (B11 * B22 - B12 * B12) - B01 * (B01 * B22 - B12 * B02) + B02 * (B01 * B12 - B11 * B02));
  r = fmin(1.0, fmax(-1.0, r));
  const double phi = acos(r) / 3.0;
  const double e1 = q + 2.0 * p * cos(phi);
  const double e3 = q + 2.0 * p * cos(phi + 2.0943951023931954923);
  lmax = e1;
  lmin = e3;
}

__global__ void eq55_kernel(Ctx cx, const double* gtab, double* partials) {
  const Geo g = cx.g;
  __shared__ double sh[32];
  double mn = 1e300, mx = -1e300;
  const long long ns = g.nspec;
  const double nn = g.dirz ? (double)g.n
                           : (g.zpad ? 0.5 * g.N1 * (g.Ny ? g.Ny : g.N2) * g.N3 : (double)g.N1 * (g.Ny ? g.Ny : g.N2) * g.N3);
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < ns; b += (long long)gridDim.x * blockDim.x) {
    if (b == 0 && !g.dirz && !g.zpad && g.ky0 == 0 && !g.dmask) continue;  // periodic: G_hat(0) = 0 shares the null space
    if (g.zpad && ((b / g.N2) & (g.N3 - 1)) == 0) continue;  // slab Dirichlet z: index 0 is not a sine mode
    if (g.dir3 && ((b & (g.N1 - 1)) == 0 || ((b / g.N1) & (g.N2 - 1)) == 0 || b / ((long long)g.N1 * g.N2) == 0))
      continue;  // all-Dirichlet: index-0 entries are not modes
    if (g.dim == 2 && g.dmask == 3 && ((b % g.N1) == 0 || (b / g.N1) == 0)) continue;
    if (g.dim == 2 && g.dmask == 2 && (b % g.N2) == 0) continue;
    double lo, hi;
    if (g.c == 1) {
      lo = hi = gtab[b] * nn;
    } else if (g.c == 2) {
      const double a = gtab[b] * nn, c = gtab[ns + b] * nn, o = gtab[2 * ns + b] * nn;
      const double m = 0.5 * (a + c), r = sqrt(0.25 * (a - c) * (a - c) + o * o);
      lo = m - r;
      hi = m + r;
    } else {
      eig_sym3(gtab[b] * nn, gtab[ns + b] * nn, gtab[3 * ns + b] * nn, gtab[2 * ns + b] * nn, gtab[4 * ns + b] * nn,
               gtab[5 * ns + b] * nn, lo, hi);
    }
    mn = fmin(mn, lo);
    mx = fmax(mx, hi);
  }
  const double bmx = block_reduce<true>(mx, sh);
  __syncthreads();
  const double bmn = -block_reduce<true>(-mn, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bmn;
    partials[gridDim.x + blockIdx.x] = bmx;
  }
}

// Fixed-order combine of the per-CTA partials of one reduction slot and the CG scalar step
// that consumes it (Alg 2 l.3 / l.7-8 / l.10); one CTA per load case.
constexpr int SC_T = 1024;
__global__ void __launch_bounds__(SC_T) scalar_kernel(Ctx cx, int slot, int nblk, int mode) {
  __shared__ double sh[32];
  const int load = blockIdx.x;
  LoadState* st = cx.st + load;
  if (mode == CG && !st->active) return;
  const double* part = red_partials(cx.sc, slot, load);
  const bool mx = slot == RED_RNORM;
  // fixed-order combine (deterministic); 8 independent loads in flight per thread, since the
  // partials come from L2 and a dependent chain of them is pure latency
  double acc = 0.0;  // identity of both: ||r||_inf >= 0, sums
  for (int i0 = threadIdx.x; i0 < nblk; i0 += 8 * SC_T) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * SC_T;
      v[u] = i < nblk ? __ldcg(part + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = mx ? fmax(acc, v[u]) : acc + v[u];
  }
  const double tot = mx ? block_reduce<true>(acc, sh) : block_reduce<false>(acc, sh);
  if (threadIdx.x == 0) {
    if (mode == CG) {
      if (slot == RED_RNORM) scalar_after_rnorm(st, tot, cx.hist, cx.hist_stride, load);
      else if (slot == RED_GAMMA) scalar_after_gamma(st, tot, cx.hist, cx.hist_stride, load);
      else scalar_after_dp(st, tot, cx.hist, cx.hist_stride, load);
    } else {
      cx.sc.results[slot * kMaxRhs + load] = tot;
    }
  }
}

int launch_scalar(const Ctx& cx, int slot, int mode, cudaStream_t s) {
  const Geo& g = cx.g;
  int nblk;
  if (slot == RED_RNORM) {
    nblk = g.c * g.P3 * g.N2 / 8;
  } else if (slot == RED_GAMMA) {
    nblk = gpass_nblk(g);
  } else {
    if (g.dim == 3 && g.c == 1) {
      const int TX = g.N1 < 32 ? g.N1 : 32, ZC = g.KZC;
      const int TY = (TX == 32 && k_nr(g) == 4) ? 16 : KT_TY;
      nblk = (g.N1 / TX) * (g.N2 / TY) * ((g.P3 + ZC - 1) / ZC);
    } else if (g.dim == 3) {
      nblk = kp_elastic_modal_nblk(g);
    } else {
      nblk = (int)((g.n + 255) / 256);
    }
  }
  scalar_kernel<<<g.nrhs, SC_T, 0, s>>>(cx, slot, nblk, mode);
  return 1;
}

int launch_scalar_n(const Ctx& cx, int slot, int mode, int nblk, cudaStream_t s) {
  scalar_kernel<<<cx.g.nrhs, SC_T, 0, s>>>(cx, slot, nblk, mode);
  return 1;
}

// Device-side loop control of the CUDA-graph WHILE node: keep iterating while any load case
// is active (and below a safety cap on body executions).
__global__ void loop_ctl_kernel(cudaGraphConditionalHandle h, const LoadState* st, int nrhs, int* counter, int cap) {
  int any = 0;
  for (int l = 0; l < nrhs; ++l) any |= st[l].active;
  const int c = ++(*counter);
  if (!any || c >= cap) {
    *counter = 0;
    cudaGraphSetConditional(h, 0u);
  } else {
    cudaGraphSetConditional(h, 1u);
  }
}

int launch_loop_ctl(cudaGraphConditionalHandle h, const LoadState* st, int nrhs, int* counter, int cap, cudaStream_t s) {
  loop_ctl_kernel<<<1, 1, 0, s>>>(h, st, nrhs, counter, cap);
  return 1;
}

__global__ void zero_kernel(double* x, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = 0.0;
}

// ============================================================================== launchers
template <class F>
static int dispatch_pow2(int L, F&& f) {
  switch (L) {
    case 4: return f(std::integral_constant<int, 4>{});
    case 8: return f(std::integral_constant<int, 8>{});
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

template <class K>
static void set_smem(K kernel, int bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int launch_xfwd(const Ctx& cx, int mode, const double* src, cudaStream_t s, int b0, int nb) {
  const Geo& g = cx.g;
  if (g.N1 == 256) {
    const dim3 grid(nb > 0 ? (unsigned)nb : (unsigned)((long long)g.c * g.P3 * g.N2 / 8), g.nrhs);
    if (mode == CG) xfwd256_kernel<CG><<<grid, 128, 0, s>>>(cx, src, b0);
    else if (mode == PLAIN) xfwd256_kernel<PLAIN><<<grid, 128, 0, s>>>(cx, src, b0);
    else xfwd256_kernel<STANDALONE><<<grid, 128, 0, s>>>(cx, src, b0);
    return 1;
  }
  if (g.N1 == 512) {
    const dim3 grid(nb > 0 ? (unsigned)nb : (unsigned)((long long)g.c * g.P3 * g.N2 / 8), g.nrhs);
    if (mode == CG) xfwd512_kernel<CG><<<grid, 128, 0, s>>>(cx, src, b0);
    else if (mode == PLAIN) xfwd512_kernel<PLAIN><<<grid, 128, 0, s>>>(cx, src, b0);
    else xfwd512_kernel<STANDALONE><<<grid, 128, 0, s>>>(cx, src, b0);
    return 1;
  }
  return dispatch_pow2(g.M, [&](auto Lc) {
    constexpr int M = decltype(Lc)::value;
    const dim3 grid(nb > 0 ? (unsigned)nb : (unsigned)((long long)g.c * g.P3 * g.N2 / 8), g.nrhs);
    const int sm = xsmem_bytes<M, false>();
    if (mode == CG) {
      auto k = xfwd_kernel<M, CG>;
      set_smem(k, sm);
      k<<<grid, fft_threads(M), sm, s>>>(cx, src, b0);
    } else if (mode == PLAIN) {
      auto k = xfwd_kernel<M, PLAIN>;
      set_smem(k, sm);
      k<<<grid, fft_threads(M), sm, s>>>(cx, src, b0);
    } else {
      auto k = xfwd_kernel<M, STANDALONE>;
      set_smem(k, sm);
      k<<<grid, fft_threads(M), sm, s>>>(cx, src, b0);
    }
    return 1;
  });
}

int launch_xinv(const Ctx& cx, int mode, double* dst, cudaStream_t s, int b0, int nb) {
  const Geo& g = cx.g;
  if (g.N1 == 512) {
    const dim3 grid(nb > 0 ? (unsigned)nb : (unsigned)((long long)g.c * g.P3 * g.N2 / 8), g.nrhs);
    if (mode == CG) xinv512_kernel<CG><<<grid, 128, 0, s>>>(cx, dst, b0);
    else if (mode == PLAIN) xinv512_kernel<PLAIN><<<grid, 128, 0, s>>>(cx, dst, b0);
    else xinv512_kernel<STANDALONE><<<grid, 128, 0, s>>>(cx, dst, b0);
    return 1;
  }
  return dispatch_pow2(g.M, [&](auto Lc) {
    constexpr int M = decltype(Lc)::value;
    const dim3 grid(nb > 0 ? (unsigned)nb : (unsigned)((long long)g.c * g.P3 * g.N2 / 8), g.nrhs);
    const int sm = xsmem_bytes<M, true>();
    if (mode == CG) {
      auto k = xinv_kernel<M, CG>;
      set_smem(k, sm);
      k<<<grid, fft_threads(M), sm, s>>>(cx, dst, b0);
    } else if (mode == PLAIN) {
      auto k = xinv_kernel<M, PLAIN>;
      set_smem(k, sm);
      k<<<grid, fft_threads(M), sm, s>>>(cx, dst, b0);
    } else {
      auto k = xinv_kernel<M, STANDALONE>;
      set_smem(k, sm);
      k<<<grid, fft_threads(M), sm, s>>>(cx, dst, b0);
    }
    return 1;
  });
}

int launch_ypass(const Ctx& cx, int mode, bool inverse, cudaStream_t s, int z0, int zc) {
  const Geo& g = cx.g;
  if (zc > 0 && ((zc | z0) & 7)) return -1;
  if (g.N2 == 512 && !(zc > 0 && (zc % Y5_ROWS))) {
    const long long nrows = zc > 0 ? (long long)g.c * g.H1 * zc : (long long)g.c * g.H1 * g.P3;
    const dim3 grid((unsigned)((nrows + Y5_ROWS - 1) / Y5_ROWS), g.nrhs);
    if (mode == CG) {
      if (inverse) ypass512_kernel<true, CG><<<grid, 128, 0, s>>>(cx, z0, zc);
      else ypass512_kernel<false, CG><<<grid, 128, 0, s>>>(cx, z0, zc);
    } else {
      if (inverse) ypass512_kernel<true, STANDALONE><<<grid, 128, 0, s>>>(cx, z0, zc);
      else ypass512_kernel<false, STANDALONE><<<grid, 128, 0, s>>>(cx, z0, zc);
    }
    return 1;
  }
  if (g.N2 == 256) {
    const long long nrows = zc > 0 ? (long long)g.c * g.H1 * zc : (long long)g.c * g.H1 * g.P3;
    const dim3 grid((unsigned)((nrows + YR_ROWS - 1) / YR_ROWS), g.nrhs);
    if (mode == CG) {
      if (inverse) ypass256_kernel<true, CG><<<grid, YR_ROWS * YR_R, 0, s>>>(cx, z0, zc);
      else ypass256_kernel<false, CG><<<grid, YR_ROWS * YR_R, 0, s>>>(cx, z0, zc);
    } else {
      if (inverse) ypass256_kernel<true, STANDALONE><<<grid, YR_ROWS * YR_R, 0, s>>>(cx, z0, zc);
      else ypass256_kernel<false, STANDALONE><<<grid, YR_ROWS * YR_R, 0, s>>>(cx, z0, zc);
    }
    return 1;
  }
  return dispatch_pow2(g.N2, [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    const long long nrows = zc > 0 ? (long long)g.c * g.H1 * zc : (long long)g.c * g.H1 * g.P3;
    const dim3 grid((unsigned)((nrows + 7) / 8), g.nrhs);
    const int sm = ysmem_bytes<L>();
    auto pick = [&](auto k) {
      set_smem(k, sm);
      k<<<grid, fft_threads(L), sm, s>>>(cx, z0, zc);
    };
    if (mode == CG) {
      if (inverse) pick(ypass_kernel<L, true, CG>); else pick(ypass_kernel<L, false, CG>);
    } else {
      if (inverse) pick(ypass_kernel<L, true, STANDALONE>); else pick(ypass_kernel<L, false, STANDALONE>);
    }
    return 1;
  });
}

static bool gpass_e256(const Geo& g) {
  return g.dim == 3 && !g.dirz && g.c == 3 && g.N3 == 256 && g.N2 % GE_COLS == 0;
}
static bool gpass_512(const Geo& g) {
  return g.dim == 3 && !g.dirz && g.c == 1 && g.N3 == 512 && g.N2 % G5_C == 0;
}
// CTAs of the CG-mode G pass = gamma partials per load
int gpass_nblk(const Geo& g) {
  if (g.zpad || (g.dirz && g.dim == 3)) return pencil_gmul_nblk();  // Dirichlet z: spectrum DST stage
  if (gpass512e_supported(g)) return gpass512e_nblk(g);
  if (g.dim == 3 && !g.dirz) return g.H1 * (g.N2 / (gpass_512(g) ? G5_C : (gpass_e256(g) ? GE_COLS : 8)));
  return (int)(((long long)g.H1 * g.P3 + 7) / 8);
}

int launch_gpass_peer(const Ctx& cx, cudaStream_t s) {
  const Geo& g = cx.g;
  if (g.dim != 3 || g.dirz || gpass_512(g) || gpass_e256(g) || (g.c == 1 && g.N3 == 256)) return -1;
  return dispatch_pow2(g.N3, [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    const dim3 grid((unsigned)(g.H1 * (g.N2 / 8)), g.nrhs);
    auto go = [&](auto k, int sm) {
      set_smem(k, sm);
      k<<<grid, fft_threads(L), sm, s>>>(cx);
      return 1;
    };
    if (g.c == 1) return go(gpass_z_kernel<L, 1, CG, true>, gsmem_bytes<L, 1>());
    if constexpr (gsmem_bytes<L, 3>() <= 220 * 1024) {
      return go(gpass_z_kernel<L, 3, CG, true>, gsmem_bytes<L, 3>());
    } else {
      return -1;
    }
  });
}

int launch_gpass(const Ctx& cx, int mode, cudaStream_t s) {
  const Geo& g = cx.g;
  if (mode == FWDZ) {  // forward z FFT of the half spectrum (3D periodic; training features)
    if (g.dim != 3 || g.dirz || g.dir3) return -1;
    return dispatch_pow2(g.N3, [&](auto Lc) {
      constexpr int L = decltype(Lc)::value;
      const dim3 grid((unsigned)(g.H1 * (g.N2 / 8)), g.nrhs);
      auto go = [&](auto k, int sm) {
        set_smem(k, sm);
        k<<<grid, fft_threads(L), sm, s>>>(cx);
        return 1;
      };
      if (g.c == 1) return go(gpass_z_kernel<L, 1, FWDZ>, gsmem_tile_bytes<L, 1>());
      if constexpr (gsmem_tile_bytes<L, 3>() <= 220 * 1024) {
        return go(gpass_z_kernel<L, 3, FWDZ>, gsmem_tile_bytes<L, 3>());
      } else {
        return -1;
      }
    });
  }
  if (g.dim == 3 && !g.dirz && g.c == 1 && g.N3 == 256) {
    if (gpass256t_supported(g) && launch_gpass256t(cx, mode, s) > 0) return 1;  // TMA-streamed persistent kernel
    const dim3 grid((unsigned)(g.H1 * (g.N2 / 8) * g.nrhs));
    constexpr int sm = (8 * GR_CS + 256) * 16 + 256 * 8 * 8;
    if (mode == CG) {
      set_smem(gpass256_kernel<CG>, sm);
      gpass256_kernel<CG><<<grid, 8 * YR_R, sm, s>>>(cx);
    } else {
      set_smem(gpass256_kernel<STANDALONE>, sm);
      gpass256_kernel<STANDALONE><<<grid, 8 * YR_R, sm, s>>>(cx);
    }
    return 1;
  }
  if (mode != FWDZ && gpass_512(g)) {
    const dim3 grid((unsigned)(g.H1 * (g.N2 / G5_C)), g.nrhs);
    if (mode == CG) {
      set_smem(gpass512_kernel<CG>, gpass512_smem);
      gpass512_kernel<CG><<<grid, G5_T, gpass512_smem, s>>>(cx);
    } else {
      set_smem(gpass512_kernel<STANDALONE>, gpass512_smem);
      gpass512_kernel<STANDALONE><<<grid, G5_T, gpass512_smem, s>>>(cx);
    }
    return 1;
  }
  if (mode != FWDZ && gpass_e256(g)) {
    const dim3 grid((unsigned)(g.H1 * (g.N2 / GE_COLS)), g.nrhs);
    if (mode == CG) {
      set_smem(gpass256e_kernel<CG>, gpass256e_smem);
      gpass256e_kernel<CG><<<grid, 3 * GE_COLS * YR_R, gpass256e_smem, s>>>(cx);
    } else {
      set_smem(gpass256e_kernel<STANDALONE>, gpass256e_smem);
      gpass256e_kernel<STANDALONE><<<grid, 3 * GE_COLS * YR_R, gpass256e_smem, s>>>(cx);
    }
    return 1;
  }
  if (mode != FWDZ && gpass512e_supported(g)) return launch_gpass512e(cx, mode, s);
  if (g.dim == 3 && !g.dirz) {
    return dispatch_pow2(g.N3, [&](auto Lc) {
      constexpr int L = decltype(Lc)::value;
      const dim3 grid((unsigned)(g.H1 * (g.N2 / 8)), g.nrhs);
      auto go = [&](auto k, int sm) {
        set_smem(k, sm);
        k<<<grid, fft_threads(L), sm, s>>>(cx);
        return 1;
      };
      if (g.c == 1) {
        return mode == CG ? go(gpass_z_kernel<L, 1, CG>, gsmem_bytes<L, 1>())
                          : go(gpass_z_kernel<L, 1, STANDALONE>, gsmem_bytes<L, 1>());
      }
      if constexpr (gsmem_bytes<L, 3>() <= 220 * 1024) {
        return mode == CG ? go(gpass_z_kernel<L, 3, CG>, gsmem_bytes<L, 3>())
                          : go(gpass_z_kernel<L, 3, STANDALONE>, gsmem_bytes<L, 3>());
      } else {
        return -1;
      }
    });
  }
  return dispatch_pow2(g.N2, [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    const dim3 grid((unsigned)(((long long)g.H1 * g.P3 + 7) / 8), g.nrhs);
    auto go = [&](auto k, int sm) {
      set_smem(k, sm);
      k<<<grid, fft_threads(L), sm, s>>>(cx);
      return 1;
    };
    if (g.c == 1)
      return mode == CG ? go(gpass_y2d_kernel<L, 1, CG>, gsmem_bytes<L, 1>())
                        : go(gpass_y2d_kernel<L, 1, STANDALONE>, gsmem_bytes<L, 1>());
    if (g.c == 2)
      return mode == CG ? go(gpass_y2d_kernel<L, 2, CG>, gsmem_bytes<L, 2>())
                        : go(gpass_y2d_kernel<L, 2, STANDALONE>, gsmem_bytes<L, 2>());
    if constexpr (gsmem_bytes<L, 3>() <= 220 * 1024) {
      return mode == CG ? go(gpass_y2d_kernel<L, 3, CG>, gsmem_bytes<L, 3>())
                        : go(gpass_y2d_kernel<L, 3, STANDALONE>, gsmem_bytes<L, 3>());
    } else {
      return -1;
    }
  });
}

int launch_kapply(const Ctx& cx, int mode, const double* src, double* dst, cudaStream_t s, int zc0, int nzl) {
  const Geo& g = cx.g;
  if (g.dim == 3 && g.c == 1) {
    const int TX = g.N1 < 32 ? g.N1 : 32;
    const int ZC = g.KZC;
    const int nzc = (g.P3 + ZC - 1) / ZC;
    if (nzl <= 0) {
      zc0 = 0;
      nzl = nzc;
    } else if (TX != 32) {
      return -1;  // z-chunk ranges: production kernel only
    }
    const int sm = (KT_RING * 10 * (TX + 2) + 4 * 9 * (TX + 1)) * (int)sizeof(double);
    const dim3 grid(g.N1 / TX, g.N2 / KT_TY, nzl * g.nrhs);
    if (g.dirz && TX != 32) return -1;  // mixed BC: production kernel only (N1 >= 32)
    auto go = [&](auto kern, int tpb) {
      set_smem(kern, sm);
      kern<<<grid, tpb, sm, s>>>(cx, mode, src, dst, ZC);
    };
    if (g.halo && !(TX == 32 && k_nr(g) == 4)) {
      return -1;  // slab halos: the NR = 4 kernel only
    } else if (TX == 32 && k_nr(g) == 4) {
      const dim3 grid4(g.N1 / 32, g.N2 / 16, nzl * g.nrhs);
      const int sm4 = KT_RING * (18 * KR2_DW * (int)sizeof(double) + 17 * KR2_PW);
      auto k4 = g.halo ? kp_thermal3d_rn_kernel<4, true, false>
                       : (g.dir3 ? kp_thermal3d_rn_kernel<4, false, true> : kp_thermal3d_rn_kernel<4, false, false>);
      set_smem(k4, sm4);
      k4<<<grid4, 128, sm4, s>>>(cx, mode, src, dst, ZC, zc0, nzl);
    } else if (TX == 32) {
      const int sm2 = KT_RING * (KR2_DPL * (int)sizeof(double) + KR2_PHS);
      auto k2 = kp_thermal3d_r2_kernel<32, 4>;
      set_smem(k2, sm2);
      k2<<<grid, 128, sm2, s>>>(cx, mode, src, dst, ZC, zc0, nzl);
    }
    else if (TX == 16) go(kp_thermal3d_kernel<16>, 128);
    else go(kp_thermal3d_kernel<8>, 64);
    return 1;
  }
  if (g.dim == 2 && g.c == 1) {
    const dim3 grid((unsigned)((g.n + 255) / 256), g.nrhs);
    kp_thermal2d_kernel<<<grid, 256, 0, s>>>(cx, mode, src, dst);
    return 1;
  }
  if (g.dim == 3) {
    return launch_kp_elastic_modal(cx, mode, src, dst, s);
  }
  const dim3 grid((unsigned)((g.n + 255) / 256), g.nrhs);
  kp_elastic2d_kernel<<<grid, 256, 0, s>>>(cx, mode, src, dst);
  return 1;
}

int launch_rhs(const Ctx& cx, const LoadParams& lp, double* f, cudaStream_t s) {
  long long nb = (cx.g.n + 255) / 256;
  if (nb > 148 * 8) nb = 148 * 8;
  rhs_kernel<<<(unsigned)nb, 256, 0, s>>>(cx, lp, f);
  return 1;
}

int launch_finalize(const Ctx& cx, cudaStream_t s) {
  const long long cnt = (long long)cx.g.c * cx.g.n;
  long long nb = (cnt + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  finalize_kernel<<<dim3((unsigned)nb, cx.g.nrhs), 256, 0, s>>>(cx);
  return 1;
}

int launch_mean_removal(const Ctx& cx, const double* u, double* out, double* scratch, cudaStream_t s) {
  const Geo& g = cx.g;
  const int nlc = g.nrhs * g.c;
  const int nblk = 148 * 2;
  double* partials = scratch;            // [nlc][nblk]
  double* means = scratch + (long long)nlc * nblk;
  mean_partial_kernel<<<dim3(nblk, nlc), 256, 0, s>>>(u, g.n, partials, nblk);
  mean_combine_kernel<<<nlc, 256, 0, s>>>(partials, nblk, g.n, means);
  long long nb = (g.n + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  mean_subtract_kernel<<<dim3((unsigned)nb, nlc), 256, 0, s>>>(u, out, g.n, means);
  return 3;
}

int launch_effective(const Ctx& cx, const LoadParams& lp, const double* u, double* partials, int* nblocks_out,
                     cudaStream_t s) {
  const int nblk = 148 * 4;
  const int nacc = cx.g.nrhs * cx.g.nrhs + 1;
  auto pick = [&](auto nlc) {
    constexpr int NL = decltype(nlc)::value;
    if (cx.g.c == 1) effective_n_kernel<NL, 1><<<nblk, EFF_T, 0, s>>>(cx, lp, u, partials);
    else if (cx.g.c == 2) effective_n_kernel<NL, 2><<<nblk, EFF_T, 0, s>>>(cx, lp, u, partials);
    else effective_n_kernel<NL, 3><<<nblk, EFF_T, 0, s>>>(cx, lp, u, partials);
  };
  switch (cx.g.nrhs) {
    case 1: pick(std::integral_constant<int, 1>{}); break;
    case 2: pick(std::integral_constant<int, 2>{}); break;
    case 3: pick(std::integral_constant<int, 3>{}); break;
    case 4: pick(std::integral_constant<int, 4>{}); break;
    case 5: pick(std::integral_constant<int, 5>{}); break;
    case 6: pick(std::integral_constant<int, 6>{}); break;
    case 7: pick(std::integral_constant<int, 7>{}); break;
    default: pick(std::integral_constant<int, 8>{}); break;
  }
  combine_rows_kernel<<<nacc, 256, 0, s>>>(partials, nblk, partials + (long long)nacc * nblk);
  *nblocks_out = nblk;
  return 2;
}

int launch_build_symbol(const Ctx& cx, double* gtab, double ref0, double ref1, unsigned long long seed, double amp,
                        cudaStream_t s) {
  build_symbol_kernel<<<(unsigned)((cx.g.nspec + 255) / 256), 256, 0, s>>>(cx, gtab, ref0, ref1, seed, amp);
  return 1;
}

int launch_eq55(const Ctx& cx, const double* gtab, double* partials, int* nblocks_out, cudaStream_t s) {
  const int nblk = 148 * 2;
  eq55_kernel<<<nblk, 256, 0, s>>>(cx, gtab, partials);
  *nblocks_out = nblk;
  return 1;
}

int launch_zero(double* x, long long n, cudaStream_t s) {
  long long nb = (n + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  zero_kernel<<<(unsigned)nb, 256, 0, s>>>(x, n);
  return 1;
}

int blocks_needed_max(const Geo& g) {
  long long m = (long long)g.c * g.N3 * g.N2 / 8;                // x passes
  if (g.zpad || g.dirz) m = m > pencil_gmul_nblk() ? m : pencil_gmul_nblk();  // Dirichlet-z gamma partials
  if (g.dim == 3) m = m > (long long)g.H1 * (g.N2 / 4) ? m : (long long)g.H1 * (g.N2 / 4);  // G pass
  else m = m > (g.H1 + 7) / 8 ? m : (g.H1 + 7) / 8;
  if (g.dirz) {  // DST pass grid
    const long long a = (long long)g.c * g.N2 * (g.N1 / 16);
    m = m > a ? m : a;
    const long long b2 = ((long long)g.H1 * g.P3 + 7) / 8;
    m = m > b2 ? m : b2;
  }
  long long kb;
  if (g.dim == 3 && g.c == 1) {
    const int TX = g.N1 < 32 ? g.N1 : 32, ZC = g.KZC;
    kb = (long long)(g.N1 / TX) * (g.N2 / KT_TY) * ((g.P3 + ZC - 1) / ZC);
  } else if (g.dim == 3) {
    kb = kp_elastic_modal_nblk(g);
  } else {
    kb = (g.n + 255) / 256;
  }
  // grid-stride passes of the baseline preconditioners and the Dirichlet dot (precond.cu,
  // dirichlet.cu: up to 148 x 8 CTAs): a preconditioner can be switched on any handle
  const long long jb = jacobi_nblk(g);
  kb = kb > jb ? kb : jb;
  return (int)(m > kb ? m : kb);
}

}  // namespace uno
