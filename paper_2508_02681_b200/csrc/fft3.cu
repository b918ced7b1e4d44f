// fft3.cu — the 3-pass ("four-step") schedule of the UNO apply for 3D grids.
//
// The y transform (length N2 = NA*NB, y = y_a + NA*y_b, k_y = k_b + NB*k_a) is split
// between the x pass and the z pass (decimation in time):
//   A[y_a, k_b]   = w_N2^{y_a k_b} * sum_{y_b} x[y_a + NA y_b] w_NB^{y_b k_b}        (F1)
//   X[k_b + NB k_a] = sum_{y_a} A[y_a, k_b] w_NA^{y_a k_a}                           (F2)
// so one pass over the spectrum disappears on each side:
//   F1 f1_kernel:  r -= alpha p ; ||r||_inf ; x R2C of NB rows ; NB-point DFT across them
//   F2 f2_kernel:  NA-point DFT along y_a ; z FFT ; s_hat = G_hat r_hat ; gamma_1 ; inverses
//   F3 f3_kernel:  inverse of F1 ; x C2R ; d = s + beta d ; u += alpha d_old
// (Alg 2 l.3-12; the operator is exactly T^H Q T of Eq 48 — only the order of the
// butterflies differs from the 5-pass schedule in kernels.cu.)
// Spectrum layout for this schedule: [nrhs][c][kx][k_b][kz][k_a]  (F2 reads one contiguous
// NA x N3 block per (kx, k_b)); the tabulated symbol uses the same layout.
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "dev_common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

#ifndef UNO_F1R_MINB
#define UNO_F1R_MINB 2
#endif

namespace uno {

template <int M, int NB>
__host__ __device__ constexpr int f1_stage() {
  return (NB * M > (M + 1) * (NB + 1)) ? NB * M : (M + 1) * (NB + 1);
}
template <int M, int NB>
__host__ __device__ constexpr int f3_stage() {
  return (2 * NB * M > (M + 1) * (NB + 1)) ? 2 * NB * M : (M + 1) * (NB + 1);
}
template <int M, int NB, bool INV>
__host__ __device__ constexpr int f13_smem_elems() {  // + NB twiddles w_N2^{y_a k_b} + NB/2 w_NB^r
  return NB * M + (INV ? f3_stage<M, NB>() : f1_stage<M, NB>()) + M + (M + 1) + NB + NB / 2;
}

// resident CTAs per SM the shared-memory footprint allows (1 KB driver reserve per CTA), asked of
// ptxas through __launch_bounds__ so registers do not become the tighter limit
template <int M, int NB, bool INV>
__host__ __device__ constexpr int f13_minb() {
  return (f13_smem_elems<M, NB, INV>() * 16 + 1024) * 3 <= 228 * 1024   ? 3
         : (f13_smem_elems<M, NB, INV>() * 16 + 1024) * 2 <= 228 * 1024 ? 2
                                                                       : 1;
}

// ------------------------------------------------------------------------------------- F1
template <int M, int NB, int MODE>
__global__ void __launch_bounds__(fft_threads_nt(M, NB / 8), f13_minb<M, NB, false>()) f1_kernel(Ctx cx, const double* __restrict__ src) {
  constexpr int NT = NB / 8;
  constexpr int T = fft_threads_nt(M, NT);
  constexpr int H1 = M + 1;
  constexpr int XS = NB + 1;  // padded row stride of the X[kx][y_b] buffer (bank-conflict free)
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE == CG && !st->active) return;
  extern __shared__ double2 smem[];
  double2* tiles = smem;                        // NT tiles of 8 rows x M
  double2* stage = tiles + NB * M;              // p rows, later X[kx][y_b]
  double2* tw = stage + f1_stage<M, NB>();      // M
  double2* twp = tw + M;                        // M + 1
  double2* twa = twp + H1;                      // NB: w_N2^{y_a k_b}
  double2* twb = twa + NB;                      // NB/2: w_NB^r
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int NA = g.NA, N2 = g.N2, N1 = g.N1;
  const int ya = blockIdx.x % NA;
  const int zc = blockIdx.x / NA;
  const int z = zc % g.N3, comp = zc / g.N3;
  const long long vbase = (long long)load * g.c * g.n + (long long)comp * g.n + (long long)z * N2 * N1;
  bool upd = false;
  double alpha = 0.0;
  if (MODE == CG) {
    upd = st->iters > 0;
    alpha = st->alpha;
  }
#pragma unroll
  for (int i = 0; i < (NB * M + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < NB * M) {
      const int r = e / M, j = e & (M - 1);
      const long long off = vbase + (long long)(ya + NA * r) * N1 + 2 * j;
      cp_async16(&tiles[(r >> 3) * 8 * M + tidx(j, r & 7)], src + off);
      if (MODE == CG && upd) cp_async16(&stage[e], cx.p + off);
    }
  }
  cp_commit();
  for (int i = t; i < M; i += T) tw[i] = cx.tw.x[i];
  for (int i = t; i <= M; i += T) twp[i] = cx.tw.xpost[i];
  if (t < NB) twa[t] = cx.tw.y[ya * t];
  if (t < NB / 2) twb[t] = cx.tw.y[t * NA];
  cp_wait<0>();
  __syncthreads();
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < (NB * M + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < NB * M) {
      const int r = e / M, j = e & (M - 1);
      const int ti = (r >> 3) * 8 * M + tidx(j, r & 7);
      double2 v = tiles[ti];
      if (MODE == CG && upd) {  // r <- r - alpha p   (Alg 2 l.11)
        const double2 pv = stage[e];
        v.x = fma(-alpha, pv.x, v.x);
        v.y = fma(-alpha, pv.y, v.y);
        *reinterpret_cast<double2*>(cx.r + vbase + (long long)(ya + NA * r) * N1 + 2 * j) = v;
        tiles[ti] = v;
      }
      mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
  }
  __syncthreads();
  fft_tiles<M, NT, false>(tiles, tw);
  // R2C post-processing of every row into X[kx][y_b]
#pragma unroll
  for (int i = 0; i < ((M / 2 + 1) * NB + T - 1) / T; ++i) {
    const int it = t + i * T;
    if (it < (M / 2 + 1) * NB) {
      const int r = it % NB, k = it / NB;
      const double2* tq = tiles + (r >> 3) * 8 * M;
      const double2 a = tq[tidx(k, r & 7)];
      const double2 b = cconj(tq[tidx((M - k) & (M - 1), r & 7)]);
      const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
      const double2 O = mul_mi(make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y)));
      stage[k * XS + r] = cadd(E, cmul(twp[k], O));
      if (k != M - k) stage[(M - k) * XS + r] = cadd(cconj(E), cmul(twp[M - k], cconj(O)));
    }
  }
  __syncthreads();
  // NB-point DFT across the rows (y_b -> k_b), twiddle w_N2^{y_a k_b}, scatter to [kx][k_b][z][y_a]
  double2* out = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * NA + ya;
  const long long kbstride = (long long)g.N3 * NA;
  for (int it = t; it < 2 * H1; it += T) {
    const int kx = it >> 1, h = it & 1;
    double2 v[NB], o[NB / 2];
#pragma unroll
    for (int r = 0; r < NB; ++r) v[r] = stage[kx * XS + r];
    dft_half<NB, false>(v, h, twb, o);
#pragma unroll
    for (int m = 0; m < NB / 2; ++m) {
      const int kb = 2 * m + h;
      out[((long long)kx * NB + kb) * kbstride] = kb ? cmul(o[m], twa[kb]) : o[m];
    }
  }
  if (MODE == CG) {
    double tot;
    if (grid_reduce<true>(mx, red_partials(cx.sc, RED_RNORM, load), red_counter(cx.sc, RED_RNORM, load), gridDim.x,
                          blockIdx.x, &tot, red_sh)) {
      if (threadIdx.x == 0) scalar_after_rnorm(st, tot, cx.hist, cx.hist_stride, load);
    }
  }
}

// ------------------------------------------------------------------------------------- F3
template <int M, int NB, int MODE>
__global__ void __launch_bounds__(fft_threads_nt(M, NB / 8), f13_minb<M, NB, true>()) f3_kernel(Ctx cx, double* __restrict__ dst) {
  constexpr int NT = NB / 8;
  constexpr int T = fft_threads_nt(M, NT);
  constexpr int H1 = M + 1;
  constexpr int XS = NB + 1;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE == CG && !st->active) return;
  extern __shared__ double2 smem[];
  double2* tiles = smem;
  double2* stage = tiles + NB * M;              // X[kx][k_b], later d rows | u rows
  double2* tw = stage + f3_stage<M, NB>();
  double2* twp = tw + M;
  double2* twa = twp + H1;  // NB: w_N2^{y_a k_b}
  double2* twb = twa + NB;  // NB/2: w_NB^r
  const int t = threadIdx.x;
  const int NA = g.NA, N2 = g.N2, N1 = g.N1;
  const int ya = blockIdx.x % NA;
  const int zc = blockIdx.x / NA;
  const int z = zc % g.N3, comp = zc / g.N3;
  const double2* in = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * NA + ya;
  const long long kbstride = (long long)g.N3 * NA;
#pragma unroll
  for (int i = 0; i < (H1 * NB + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < H1 * NB) cp_async16(&stage[(e / NB) * XS + (e % NB)], in + (long long)e * kbstride);
  }
  cp_commit();
  for (int i = t; i < M; i += T) tw[i] = cx.tw.x[i];
  for (int i = t; i <= M; i += T) twp[i] = cx.tw.xpost[i];
  if (t < NB) twa[t] = cx.tw.y[ya * t];
  if (t < NB / 2) twb[t] = cx.tw.y[t * NA];
  cp_wait<0>();
  __syncthreads();
  // conj twiddle + inverse NB-point DFT (k_b -> y_b), in place; two threads per kx (outputs
  // y_b = 2m + h), so every round reads all inputs before anyone writes
#pragma unroll 1
  for (int i = 0; i < (2 * H1 + T - 1) / T; ++i) {
    const int it = t + i * T;
    const int kx = it >> 1, h = it & 1;
    const bool act = it < 2 * H1;
    double2 o[NB / 2];
    if (act) {
      double2 v[NB];
#pragma unroll
      for (int kb = 0; kb < NB; ++kb) {
        const double2 a = stage[kx * XS + kb];
        v[kb] = kb ? cmul(a, cconj(twa[kb])) : a;
      }
      dft_half<NB, true>(v, h, twb, o);
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int m = 0; m < NB / 2; ++m) stage[kx * XS + 2 * m + h] = o[m];
    }
  }
  __syncthreads();
  // C2R pre-processing of each row r into the x tiles
#pragma unroll
  for (int i = 0; i < ((M / 2 + 1) * NB + T - 1) / T; ++i) {
    const int it = t + i * T;
    if (it < (M / 2 + 1) * NB) {
      const int r = it % NB, k = it / NB;
      double2* tq = tiles + (r >> 3) * 8 * M;
      const int c = r & 7;
      if (k == 0) {
        const double X0 = stage[r].x, XM = stage[M * XS + r].x;
        tq[tidx(0, c)] = make_double2(X0 + XM, X0 - XM);
      } else {
        const double2 a = stage[k * XS + r];
        const double2 bm = stage[(M - k) * XS + r];
        const double2 b = cconj(bm);
        const double2 E = cadd(a, b);
        const double2 O = cmul(csub(a, b), cconj(twp[k]));
        tq[tidx(k, c)] = cadd(E, mul_pi(O));
        if (k != M - k) {
          const double2 a2 = bm, b2 = cconj(a);
          const double2 E2 = cadd(a2, b2);
          const double2 O2 = cmul(csub(a2, b2), cconj(twp[M - k]));
          tq[tidx(M - k, c)] = cadd(E2, mul_pi(O2));
        }
      }
    }
  }
  __syncthreads();
  const long long vbase = (long long)load * g.c * g.n + (long long)comp * g.n + (long long)z * N2 * N1;
  const int it0 = MODE == CG ? st->iters : 0;
  if (MODE == CG) {  // d_old and u rows land while the inverse x FFT runs
    if (it0 > 0) {
#pragma unroll
      for (int i = 0; i < (NB * M + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < NB * M) {
          const int r = e / M, j = e & (M - 1);
          const long long off = vbase + (long long)(ya + NA * r) * N1 + 2 * j;
          cp_async16(&stage[e], cx.d + off);
          cp_async16(&stage[NB * M + e], cx.u + off);
        }
      }
    }
    cp_commit();
  }
  fft_tiles<M, NT, true>(tiles, tw);
  if (MODE == CG) {
    cp_wait<0>();
    __syncthreads();
  }
  const double beta = MODE == CG ? st->beta : 0.0, alpha = MODE == CG ? st->alpha : 0.0;
#pragma unroll
  for (int i = 0; i < (NB * M + T - 1) / T; ++i) {
    const int e = t + i * T;
    if (e < NB * M) {
      const int r = e / M, j = e & (M - 1);
      const double2 s = tiles[(r >> 3) * 8 * M + tidx(j, r & 7)];
      const long long off = vbase + (long long)(ya + NA * r) * N1 + 2 * j;
      if (MODE == STANDALONE) {
        *reinterpret_cast<double2*>(dst + off) = s;
      } else if (it0 == 0) {
        *reinterpret_cast<double2*>(cx.d + off) = s;  // d = s  (Alg 2 l.2, l.8)
      } else {
        const double2 dold = stage[e];
        double2 uu = stage[NB * M + e];  // deferred u += alpha_{m-1} d_{m-1}  (Alg 2 l.12)
        uu.x = fma(alpha, dold.x, uu.x);
        uu.y = fma(alpha, dold.y, uu.y);
        *reinterpret_cast<double2*>(cx.u + off) = uu;
        *reinterpret_cast<double2*>(cx.d + off) = make_double2(fma(beta, dold.x, s.x), fma(beta, dold.y, s.y));
      }
    }
  }
}

// ------------------------------------------------------------------------------------- F2
template <int NA, int L3, int NC>
__host__ __device__ constexpr int f2_tile_elems() {
  return NC * NA * L3 + L3;  // tiles + z twiddles (double2)
}
template <int NA, int L3, int NC>
__host__ __device__ constexpr bool f2_staged() {
  return f2_tile_elems<NA, L3, NC>() * 16 + NA * L3 * (NC == 1 ? 1 : (NC == 2 ? 3 : 6)) * 8 <= 200 * 1024;
}
template <int NA, int L3, int NC>
__host__ __device__ constexpr int f2_smem_bytes() {
  return f2_tile_elems<NA, L3, NC>() * 16 + (f2_staged<NA, L3, NC>() ? NA * L3 * (NC == 1 ? 1 : (NC == 2 ? 3 : 6)) * 8 : 0);
}

template <int NA, int L3, int NC, bool INV>
__device__ __forceinline__ void row_dft(double2* const* tiles) {
  // NA-point DFT along the tile columns of each row z (columns a = 0..NA-1 over NA/8 tiles)
  for (int z = threadIdx.x; z < L3; z += blockDim.x) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double2 v[NA];
#pragma unroll
      for (int a = 0; a < NA; ++a) v[a] = tiles[q][(a >> 3) * 8 * L3 + tidx(z, a & 7)];
      dft_reg<NA, INV>(v);
#pragma unroll
      for (int a = 0; a < NA; ++a) tiles[q][(a >> 3) * 8 * L3 + tidx(z, a & 7)] = v[a];
    }
  }
}

template <int NA, int L3, int NC, int MODE>
__global__ void __launch_bounds__(fft_threads_nt(L3, NA / 8)) f2_kernel(Ctx cx) {
  constexpr int NT = NA / 8;
  constexpr int T = fft_threads_nt(L3, NT);
  constexpr int NCC = NC == 1 ? 1 : (NC == 2 ? 3 : 6);
  constexpr bool STG = f2_staged<NA, L3, NC>();
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tiles[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) tiles[q] = smem + q * NA * L3;
  double2* tw = smem + NC * NA * L3;
  double* gs = reinterpret_cast<double*>(tw + L3);
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int kxkb = blockIdx.x;
  const int kx = kxkb / g.NB;
  const long long boff = (long long)kxkb * L3 * NA;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const double2* base = cx.spec + ((long long)load * g.c + q) * g.nspec + boff;
#pragma unroll
    for (int i = 0; i < (NA * L3 + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < NA * L3) {
        const int z = e / NA, a = e % NA;
        cp_async16(&tiles[q][(a >> 3) * 8 * L3 + tidx(z, a & 7)], base + e);
      }
    }
  }
  if (STG) {
#pragma unroll
    for (int q = 0; q < NCC; ++q) {
#pragma unroll
      for (int i = 0; i < (NA * L3 + T - 1) / T; ++i) {
        const int e = t + i * T;
        if (e < NA * L3) cp_async8(&gs[q * NA * L3 + e], cx.gtab + q * g.nspec + boff + e);
      }
    }
  }
  cp_commit();
  for (int i = t; i < L3; i += T) tw[i] = cx.tw.z[i];
  cp_wait<0>();
  __syncthreads();
  row_dft<NA, L3, NC, false>(tiles);
  __syncthreads();
  const double w = parseval_w(kx, g.M);
  double part = 0.0;
  if constexpr (gconv_fusable(L3) && NC * plan_radix(L3, plan_stages(L3) - 1) <= 32) {
    // symbol multiply fused into the middle butterfly of the z FFT (fft.cuh fft_gconv)
    part = fft_gconv<L3, NT, NC>(tiles, tw, [&](int tq, int c, int kz, double2* x) {
      const int a = tq * 8 + c;
      return STG ? gmul_vals<NC>(x, gs, NA * L3, (long long)kz * NA + a, w)
                 : gmul_vals<NC>(x, cx.gtab, g.nspec, boff + (long long)kz * NA + a, w);
    });
  } else {
#pragma unroll
    for (int q = 0; q < NC; ++q) fft_tiles<L3, NT, false>(tiles[q], tw);
#pragma unroll
    for (int i = 0; i < (NA * L3 + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < NA * L3) {
        const int z = e / NA, a = e % NA;
        const int ti = (a >> 3) * 8 * L3 + tidx(z, a & 7);
        if (STG)
          part += gmul_bin<NC>(tiles, ti, gs, NA * L3, e, w);
        else
          part += gmul_bin<NC>(tiles, ti, cx.gtab, g.nspec, boff + e, w);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NC; ++q) fft_tiles<L3, NT, true>(tiles[q], tw);
  }
  row_dft<NA, L3, NC, true>(tiles);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    double2* base = cx.spec + ((long long)load * g.c + q) * g.nspec + boff;
#pragma unroll
    for (int i = 0; i < (NA * L3 + T - 1) / T; ++i) {
      const int e = t + i * T;
      if (e < NA * L3) {
        const int z = e / NA, a = e % NA;
        base[e] = tiles[q][(a >> 3) * 8 * L3 + tidx(z, a & 7)];
      }
    }
  }
  gamma_finish(cx, load, part, red_sh, MODE);
}

// F1 for N1 = 256 (M = 128), NB = NA = 16: register-direct.  Per row (16 threads) as
// xfwd256_kernel: z_j loaded straight into registers (j = n1 + 16 n2), r -= alpha p, ||r||_inf,
// DFT8 over n2 -> twiddle -> transpose T -> half DFT16 over n1 -> X[y_b][k] (swizzled); R2C
// post-processing into Y[kx][y_b]; then the NB-point DFT across the rows (two threads per kx)
// with the twiddle w_N2^{y_a k_b} and the scatter to [kx][k_b][z][y_a].
constexpr int F1R_TS = 16 * 8 * 17;        // T: 16 rows x [8][17]
constexpr int F1R_YS = 129 * 17;           // Y: [129][17] (aliases T)
constexpr int F1R_TY = F1R_TS > F1R_YS ? F1R_TS : F1R_YS;
constexpr int F1R_XS = 129;                // X row stride
__device__ __forceinline__ int f1r_swz(int k) { return k ^ (((k >> 3) & 1) << 2); }
__host__ __device__ constexpr int f1r_smem_bytes() { return (F1R_TY + 16 * F1R_XS + 128 + 129 + 16 + 8 + 8) * 16; }

template <int MODE>
__global__ void __launch_bounds__(256, UNO_F1R_MINB) f1r_kernel(Ctx cx, const double* __restrict__ src) {
  constexpr int M = 128, NB = 16, NA = 16;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  extern __shared__ double2 f1s[];
  double2* TY = f1s;                      // T rows, later Y[kx][y_b]
  double2* X = TY + F1R_TY;               // [16][129] swizzled
  double2* tw = X + 16 * F1R_XS;          // [128] w_128^m
  double2* twp = tw + M;                  // [129] w_256^k
  double2* twa = twp + M + 1;             // [16] w_N2^{y_a k_b}
  double2* twb = twa + NB;                // [8] w_16^r (across-row DFT)
  double2* tw16 = twb + 8;                // [8] w_16^r = w_128^{8r} (row FFT)
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int yb = t >> 4, l16 = t & 15;
  const int ya = blockIdx.x % NA;
  const int zc = blockIdx.x / NA;
  const int z = zc % g.N3, comp = zc / g.N3;
  const long long vrow = (long long)load * g.c * g.n + (long long)comp * g.n + (long long)z * g.N2 * g.N1 +
                         (long long)(ya + NA * yb) * g.N1;
  const double2* s2 = reinterpret_cast<const double2*>(src + vrow);
  double2 v[8];
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2) v[n2] = __ldcg(s2 + l16 + 16 * n2);
  double mx = 0.0;
  if (MODE == CG) {
    if (st->iters > 0) {  // r <- r - alpha p   (Alg 2 l.11)
      const double alpha = st->alpha;
      const double2* p2 = reinterpret_cast<const double2*>(cx.p + vrow);
      double2* r2 = reinterpret_cast<double2*>(cx.r + vrow);
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
  for (int i = t; i < M; i += 256) tw[i] = cx.tw.x[((i & 15) * (i >> 4)) & (M - 1)];  // [k1][n1]
  for (int i = t; i <= M; i += 256) twp[i] = cx.tw.xpost[i];
  if (t < NB) twa[t] = cx.tw.y[ya * t];
  if (t < 8) {
    twb[t] = cx.tw.y[t * NA];
    tw16[t] = cx.tw.x[8 * t];
  }
  __syncthreads();
  // row FFT stage 1 (thread (y_b, n1 = l16)): DFT8 over n2 -> k1, twiddle w_128^{n1 k1}
  dft_reg<8, false>(v);
#pragma unroll
  for (int k1 = 1; k1 < 8; ++k1) v[k1] = cmul(v[k1], tw[k1 * 16 + l16]);
  double2* Tr = TY + yb * (8 * 17);
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) Tr[k1 * 17 + l16] = v[k1];
  __syncthreads();
  {  // stage 2 (thread (y_b, k1, h)): outputs k2 = 2m + h of DFT16 over n1 ; X[k1 + 8 k2]
    const int k1 = l16 >> 1, h = l16 & 1;
    double2 a[16], o[8];
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) a[n1] = Tr[k1 * 17 + n1];
    dft_half<16, false>(a, h, tw16, o);
#pragma unroll
    for (int m = 0; m < 8; ++m) X[yb * F1R_XS + f1r_swz(k1 + 8 * (2 * m + h))] = o[m];
  }
  __syncthreads();
  // R2C post-processing (row y_b, bins k and M - k) -> Y[kx][y_b]
  for (int it = t; it < (M / 2 + 1) * NB; it += 256) {
    const int r = it & 15, k = it >> 4;
    const double2 a = X[r * F1R_XS + f1r_swz(k)];
    const double2 b = cconj(X[r * F1R_XS + f1r_swz((M - k) & (M - 1))]);
    const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
    const double2 O = mul_mi(make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y)));
    TY[k * 17 + r] = cadd(E, cmul(twp[k], O));
    if (k != M - k) TY[(M - k) * 17 + r] = cadd(cconj(E), cmul(twp[M - k], cconj(O)));
  }
  __syncthreads();
  // NB-point DFT across the rows (y_b -> k_b), twiddle w_N2^{y_a k_b}, scatter to [kx][k_b][z][y_a]
  double2* out = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * NA + ya;
  const long long kbstride = (long long)g.N3 * NA;
  for (int it = t; it < 2 * (M + 1); it += 256) {
    const int kx = it >> 1, h = it & 1;
    double2 a[16], o[8];
#pragma unroll
    for (int r = 0; r < 16; ++r) a[r] = TY[kx * 17 + r];
    dft_half<16, false>(a, h, twb, o);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int kb = 2 * m + h;
      __stcg(out + ((long long)kx * NB + kb) * kbstride, kb ? cmul(o[m], twa[kb]) : o[m]);
    }
  }
  if (MODE == CG) partial_write<true>(cx, RED_RNORM, load, blockIdx.x, mx, red_sh);
}

// F3 for N1 = 256 (M = 128), NB = NA = 16: register-direct inverse of F1.  The (z, y_a) column
// of the spectrum lands in Y[kx][k_b] by cp.async; conj twiddle + inverse half DFT16 across k_b
// (two threads per kx) -> X[y_b][kx]; C2R pre-processing in place; inverse row FFT as half
// DFT16 over k2 (thread (y_b, k1, h)) -> twiddle -> transpose T -> DFT8 over k1 (thread (y_b, n1))
// leaving s_j (j = n1 + 16 n2) in registers, where d = s + beta d_old and u += alpha d_old are
// applied with d_old / u loaded straight into registers.
constexpr int F3R_YS = 129 * 17;          // Y: [129][17]
constexpr int F3R_TS = 16 * 16 * 9;       // T: 16 rows x [16][9] (aliases Y)
constexpr int F3R_TY = F3R_YS > F3R_TS ? F3R_YS : F3R_TS;
__host__ __device__ constexpr int f3r_smem_bytes() { return (F3R_TY + 16 * F1R_XS + 128 + 129 + 16 + 8 + 8) * 16; }

template <int MODE>
__global__ void __launch_bounds__(256, UNO_F1R_MINB) f3r_kernel(Ctx cx, double* __restrict__ dst) {
  constexpr int M = 128, NB = 16, NA = 16;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  LoadState* st = cx.st + load;
  if (MODE != STANDALONE && !st->active) return;
  extern __shared__ double2 f3s[];
  double2* YT = f3s;                      // Y[kx][k_b], later T rows
  double2* X = YT + F3R_TY;               // [16][129] swizzled
  double2* tw = X + 16 * F1R_XS;          // [128] w_128^m
  double2* twp = tw + M;                  // [129] w_256^k
  double2* twa = twp + M + 1;             // [16] w_N2^{y_a k_b}
  double2* twb = twa + NB;                // [8] w_16^r (across-row DFT)
  double2* tw16 = twb + 8;                // [8] w_16^r = w_128^{8r} (row FFT)
  const int t = threadIdx.x;
  const int yb = t >> 4, l16 = t & 15;
  const int ya = blockIdx.x % NA;
  const int zc = blockIdx.x / NA;
  const int z = zc % g.N3, comp = zc / g.N3;
  const double2* in = cx.spec + ((long long)load * g.c + comp) * g.nspec + (long long)z * NA + ya;
  const long long kbstride = (long long)g.N3 * NA;
  for (int e = t; e < (M + 1) * NB; e += 256) cp_async16(&YT[(e >> 4) * 17 + (e & 15)], in + (long long)e * kbstride);
  cp_commit();
  for (int i = t; i < M; i += 256) tw[i] = cx.tw.x[i];
  for (int i = t; i <= M; i += 256) twp[i] = cx.tw.xpost[i];
  if (t < NB) twa[t] = cx.tw.y[ya * t];
  if (t < 8) {
    twb[t] = cx.tw.y[t * NA];
    tw16[t] = cx.tw.x[8 * t];
  }
  cp_wait<0>();
  __syncthreads();
  // conj twiddle + inverse DFT16 across k_b -> y_b = 2m + h ; X[y_b][kx]
  for (int it = t; it < 2 * (M + 1); it += 256) {
    const int kx = it >> 1, h = it & 1;
    double2 a[16], o[8];
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) {
      const double2 v = YT[kx * 17 + kb];
      a[kb] = kb ? cmul(v, cconj(twa[kb])) : v;
    }
    dft_half<16, true>(a, h, twb, o);
#pragma unroll
    for (int m = 0; m < 8; ++m) X[(2 * m + h) * F1R_XS + f1r_swz(kx)] = o[m];
  }
  __syncthreads();
  // C2R pre-processing of each row, in place (an item owns bins k and M - k)
  for (int it = t; it < (M / 2 + 1) * NB; it += 256) {
    const int r = it & 15, k = it >> 4;
    double2* Xr = X + r * F1R_XS;
    if (k == 0) {
      const double X0 = Xr[f1r_swz(0)].x, XM = Xr[f1r_swz(M)].x;
      Xr[f1r_swz(0)] = make_double2(X0 + XM, X0 - XM);
    } else {
      const double2 a = Xr[f1r_swz(k)];
      const double2 bm = Xr[f1r_swz(M - k)];
      const double2 b = cconj(bm);
      const double2 E = cadd(a, b);
      const double2 O = cmul(csub(a, b), cconj(twp[k]));
      Xr[f1r_swz(k)] = cadd(E, mul_pi(O));
      if (k != M - k) {
        const double2 a2 = bm, b2 = cconj(a);
        const double2 E2 = cadd(a2, b2);
        const double2 O2 = cmul(csub(a2, b2), cconj(twp[M - k]));
        Xr[f1r_swz(M - k)] = cadd(E2, mul_pi(O2));
      }
    }
  }
  __syncthreads();
  // inverse row FFT, step A (thread (y_b, k1, h)): half inverse DFT16 over k2 -> n1 = 2m + h,
  // twiddle conj(w_128^{n1 k1}) ; T[y_b][n1][k1]
  double2* Tr = YT + yb * (16 * 9);
  {
    const int k1 = l16 >> 1, h = l16 & 1;
    double2 a[16], o[8];
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) a[k2] = X[yb * F1R_XS + f1r_swz(k1 + 8 * k2)];
    dft_half<16, true>(a, h, tw16, o);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int n1 = 2 * m + h;
      Tr[n1 * 9 + k1] = n1 && k1 ? cmul(o[m], cconj(tw[(n1 * k1) & (M - 1)])) : o[m];
    }
  }
  // d_old, u rows straight into registers while the transpose settles
  const long long vrow = (long long)load * g.c * g.n + (long long)comp * g.n + (long long)z * g.N2 * g.N1 +
                         (long long)(ya + NA * yb) * g.N1;
  const int it0 = MODE == CG ? st->iters : 0;
  double2 dv[8], uv[8];
  if (MODE == CG && it0 > 0) {
    const double2* d2 = reinterpret_cast<const double2*>(cx.d + vrow);
    const double2* u2 = reinterpret_cast<const double2*>(cx.u + vrow);
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) {
      dv[n2] = __ldcs(d2 + l16 + 16 * n2);
      uv[n2] = __ldcs(u2 + l16 + 16 * n2);
    }
  }
  __syncthreads();
  // step B (thread (y_b, n1 = l16)): inverse DFT8 over k1 -> n2 ; s_j, j = n1 + 16 n2
  double2 v[8];
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) v[k1] = Tr[l16 * 9 + k1];
  dft_reg<8, true>(v);
  if (MODE == STANDALONE) {
    double2* o2 = reinterpret_cast<double2*>(dst + vrow);
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) __stcg(o2 + l16 + 16 * n2, v[n2]);
  } else {
    double2* d2 = reinterpret_cast<double2*>(cx.d + vrow);
    double2* u2 = reinterpret_cast<double2*>(cx.u + vrow);
    if (it0 == 0) {
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) __stcg(d2 + l16 + 16 * n2, v[n2]);  // d = s  (Alg 2 l.2, l.8)
    } else {
      const double beta = st->beta, alpha = st->alpha;
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) {
        const double2 dold = dv[n2];
        double2 uu = uv[n2];  // deferred u += alpha_{m-1} d_{m-1}  (Alg 2 l.12)
        uu.x = fma(alpha, dold.x, uu.x);
        uu.y = fma(alpha, dold.y, uu.y);
        __stcg(u2 + l16 + 16 * n2, uu);
        __stcg(d2 + l16 + 16 * n2, make_double2(fma(beta, dold.x, v[n2].x), fma(beta, dold.y, v[n2].y)));
      }
    }
  }
}

// F2 for NA = 16, N3 = 256, thermal: register-direct.  The (kx, k_b) block is [z][y_a] (64 KB).
// z: four-step 16 x 16 (thread (y_a, n1) loads z = n1 + 16 n2, DFT16, twiddle, transpose T1,
// DFT16 -> kz = k1 + 16 k2); y_a: transpose T2 -> thread kz does the NA-point DFT over y_a, the
// symbol multiply (+ Parseval partial of gamma) and its inverse in registers; then the z inverse
// mirrors the forward.  T1 / T2 alias one buffer; the block's symbol lands in shared memory by
// cp.async while the forward transforms run.
constexpr int F2R_YS = 16 * 17 + 1;    // T1 stride per y_a (odd in 16-byte units)
constexpr int F2R_TB = 16 * F2R_YS;    // T1 size (>= T2 = 256 x 17)
constexpr int F2R_GS = 18;             // symbol row stride (doubles): 16-byte aligned, odd in 16-byte units
__host__ __device__ constexpr int f2r_smem_bytes() { return (F2R_TB + 256) * 16 + 256 * F2R_GS * 8; }

template <int MODE>
__global__ void __launch_bounds__(256, 2) f2r_kernel(Ctx cx) {
  constexpr int R = 16, RP = R + 1, L3 = 256, NA = 16;
  const Geo g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 f2s[];
  double2* T = f2s;                                        // T1 [y_a][16][17] | T2 [kz][17]
  double2* tw = T + F2R_TB;                                // [256] w_256^m
  double* gs = reinterpret_cast<double*>(tw + L3);         // [kz][F2R_GS] symbol (k_a = 0..15)
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int ya = t & 15, l = t >> 4;
  const int kxkb = blockIdx.x;
  const int kx = kxkb / g.NB;
  const long long boff = (long long)kxkb * L3 * NA;
  double2* blk = cx.spec + (long long)load * g.nspec + boff;
  // symbol of the block (contiguous [kz][k_a]) -> padded rows
#pragma unroll
  for (int i = 0; i < L3 * NA / 2 / 256; ++i) {
    const int cidx = t + i * 256;  // 16-byte chunk
    const int kz = cidx >> 3, q = cidx & 7;
    cp_async16(&gs[kz * F2R_GS + 2 * q], cx.gtab + boff + 2 * cidx);
  }
  cp_commit();
  double2 v[R];
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) v[n2] = __ldcg(blk + (l + R * n2) * NA + ya);
  for (int i = t; i < L3; i += 256) tw[i] = cx.tw.z[i];
  __syncthreads();
  // z forward, stage 1 (thread (y_a, n1 = l))
  dft_reg<R, false>(v);
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) v[k1] = cmul(v[k1], tw[(l * k1) & (L3 - 1)]);
  double2* Ty = T + ya * F2R_YS;
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) Ty[k1 * RP + l] = v[k1];
  __syncthreads();
  // stage 2 (thread (y_a, k1 = l)): v[k2] = z-spectrum at kz = l + 16 k2
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) v[n1] = Ty[l * RP + n1];
  dft_reg<R, false>(v);
  __syncthreads();  // T1 reads done before T2 (aliased) is written
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) T[(l + R * k2) * RP + ya] = v[k2];
  cp_wait<0>();
  __syncthreads();
  // y_a DFT, symbol, inverse (thread kz = t)
  double part;
  {
    const int kz = t;
#pragma unroll
    for (int a = 0; a < NA; ++a) v[a] = T[kz * RP + a];
    dft_reg<NA, false>(v);  // v[k_a]: bin (kx, k_y = k_b + NB k_a, kz)
    const double w = parseval_w(kx, g.M);
    part = 0.0;
    const double* gr = gs + kz * F2R_GS;
#pragma unroll
    for (int a = 0; a < NA; ++a) part += gmul_vals<1>(&v[a], gr, 0, a, w);
    dft_reg<NA, true>(v);
#pragma unroll
    for (int a = 0; a < NA; ++a) T[kz * RP + a] = v[a];
  }
  __syncthreads();
  // z inverse: thread (y_a, k1 = l) reads kz = l + 16 k2
#pragma unroll
  for (int k2 = 0; k2 < R; ++k2) v[k2] = T[(l + R * k2) * RP + ya];
  dft_reg<R, true>(v);  // -> n1
#pragma unroll
  for (int n1 = 1; n1 < R; ++n1) v[n1] = cmul(v[n1], cconj(tw[(l * n1) & (L3 - 1)]));
  __syncthreads();  // T2 reads done before T1 (aliased) is written
#pragma unroll
  for (int n1 = 0; n1 < R; ++n1) Ty[n1 * RP + l] = v[n1];
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < R; ++k1) v[k1] = Ty[l * RP + k1];  // thread (y_a, n1 = l)
  dft_reg<R, true>(v);  // -> n2
#pragma unroll
  for (int n2 = 0; n2 < R; ++n2) __stcg(blk + (l + R * n2) * NA + ya, v[n2]);
  gamma_finish(cx, load, part, red_sh, MODE);
}

// ------------------------------------------------------------------------------------- launchers
template <class K>
static void set_smem3(K kernel, int bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <class F>
static int dispatch_m(int M, F&& f) {
  switch (M) {
    case 16: return f(std::integral_constant<int, 16>{});
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 128: return f(std::integral_constant<int, 128>{});
    case 256: return f(std::integral_constant<int, 256>{});
    default: return -1;
  }
}
template <class F>
static int dispatch_nb(int NB, F&& f) {
  switch (NB) {
    case 8: return f(std::integral_constant<int, 8>{});
    case 16: return f(std::integral_constant<int, 16>{});
    default: return -1;
  }
}

bool schedule3_supported(const Geo& g) {
  if (g.dim != 3 || g.N2 < 64 || g.N2 > 256 || g.M < 16 || g.M > 256) return false;
  if (g.N3 < 16 || g.N3 > 512) return false;
  const int NB = g.N2 >= 128 ? 16 : 8;
  const int NA = g.N2 / NB;
  if (NA != 8 && NA != 16) return false;
  // F2 tile must fit the shared memory of one CTA
  const long long bytes = ((long long)g.c * NA * g.N3 + g.N3) * 16;
  return bytes <= 200 * 1024 && (g.c == 1 || g.c == 3);
}

int launch_f1(const Ctx& cx, int mode, const double* src, cudaStream_t s) {
  const Geo& g = cx.g;
  static const bool rd = [] {
    const char* e = getenv("UNO_F1RD");
    return !(e && e[0] == '0');
  }();
  if (rd && g.N1 == 256 && g.NA == 16 && g.NB == 16) {
    const dim3 grid((unsigned)(g.NA * g.N3 * g.c), g.nrhs);
    constexpr int sm = f1r_smem_bytes();
    auto go = [&](auto k) {
      set_smem3(k, sm);
      k<<<grid, 256, sm, s>>>(cx, src);
      return 1;
    };
    return mode == CG ? go(f1r_kernel<CG>) : go(f1r_kernel<STANDALONE>);
  }
  return dispatch_m(g.M, [&](auto Mc) {
    constexpr int M = decltype(Mc)::value;
    return dispatch_nb(g.NB, [&](auto Bc) {
      constexpr int NB = decltype(Bc)::value;
      const int sm = f13_smem_elems<M, NB, false>() * 16;
      const dim3 grid((unsigned)(g.NA * g.N3 * g.c), g.nrhs);
      auto go = [&](auto k) {
        set_smem3(k, sm);
        k<<<grid, fft_threads_nt(M, NB / 8), sm, s>>>(cx, src);
        return 1;
      };
      return mode == CG ? go(f1_kernel<M, NB, CG>) : go(f1_kernel<M, NB, STANDALONE>);
    });
  });
}

int launch_f3(const Ctx& cx, int mode, double* dst, cudaStream_t s) {
  const Geo& g = cx.g;
  static const bool rd = [] {
    const char* e = getenv("UNO_F3RD");
    return !(e && e[0] == '0');
  }();
  if (rd && g.N1 == 256 && g.NA == 16 && g.NB == 16) {
    const dim3 grid((unsigned)(g.NA * g.N3 * g.c), g.nrhs);
    constexpr int sm = f3r_smem_bytes();
    auto go = [&](auto k) {
      set_smem3(k, sm);
      k<<<grid, 256, sm, s>>>(cx, dst);
      return 1;
    };
    return mode == CG ? go(f3r_kernel<CG>) : go(f3r_kernel<STANDALONE>);
  }
  return dispatch_m(g.M, [&](auto Mc) {
    constexpr int M = decltype(Mc)::value;
    return dispatch_nb(g.NB, [&](auto Bc) {
      constexpr int NB = decltype(Bc)::value;
      const int sm = f13_smem_elems<M, NB, true>() * 16;
      const dim3 grid((unsigned)(g.NA * g.N3 * g.c), g.nrhs);
      auto go = [&](auto k) {
        set_smem3(k, sm);
        k<<<grid, fft_threads_nt(M, NB / 8), sm, s>>>(cx, dst);
        return 1;
      };
      return mode == CG ? go(f3_kernel<M, NB, CG>) : go(f3_kernel<M, NB, STANDALONE>);
    });
  });
}

template <class F>
static int dispatch_l3(int L, F&& f) {
  switch (L) {
    case 16: return f(std::integral_constant<int, 16>{});
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 128: return f(std::integral_constant<int, 128>{});
    case 256: return f(std::integral_constant<int, 256>{});
    case 512: return f(std::integral_constant<int, 512>{});
    default: return -1;
  }
}

int launch_f2(const Ctx& cx, int mode, cudaStream_t s) {
  const Geo& g = cx.g;
  static const bool rd = [] {
    const char* e = getenv("UNO_F2RD");
    return !(e && e[0] == '0');
  }();
  if (rd && g.c == 1 && g.NA == 16 && g.N3 == 256) {
    const dim3 grid((unsigned)(g.H1 * g.NB), g.nrhs);
    constexpr int sm = f2r_smem_bytes();
    if (mode == CG) {
      set_smem3(f2r_kernel<CG>, sm);
      f2r_kernel<CG><<<grid, 256, sm, s>>>(cx);
    } else {
      set_smem3(f2r_kernel<STANDALONE>, sm);
      f2r_kernel<STANDALONE><<<grid, 256, sm, s>>>(cx);
    }
    return 1;
  }
  return dispatch_l3(g.N3, [&](auto Lc) {
    constexpr int L3 = decltype(Lc)::value;
    const dim3 grid((unsigned)(g.H1 * g.NB), g.nrhs);
    auto run = [&](auto Ac) {
      constexpr int NA = decltype(Ac)::value;
      auto go = [&](auto k, int sm) {
        set_smem3(k, sm);
        k<<<grid, fft_threads_nt(L3, NA / 8), sm, s>>>(cx);
        return 1;
      };
      if (g.c == 1)
        return mode == CG ? go(f2_kernel<NA, L3, 1, CG>, f2_smem_bytes<NA, L3, 1>())
                          : go(f2_kernel<NA, L3, 1, STANDALONE>, f2_smem_bytes<NA, L3, 1>());
      if constexpr (f2_smem_bytes<NA, L3, 3>() <= 220 * 1024) {
        return mode == CG ? go(f2_kernel<NA, L3, 3, CG>, f2_smem_bytes<NA, L3, 3>())
                          : go(f2_kernel<NA, L3, 3, STANDALONE>, f2_smem_bytes<NA, L3, 3>());
      } else {
        return -1;
      }
    };
    if (g.NA == 8) return run(std::integral_constant<int, 8>{});
    if (g.NA == 16) return run(std::integral_constant<int, 16>{});
    return -1;
  });
}

}  // namespace uno
