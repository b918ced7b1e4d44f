// dev_common.cuh — device helpers shared by the kernel translation units of libunocg:
// device-side CG scalar logic (Alg 2 l.3, l.7-8, l.10), deterministic grid reductions,
// cp.async wrappers and the per-frequency symbol multiply (Eq 46/49, Eq B7 order).
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace uno {

enum { ST_OK = 0, ST_BREAKDOWN = 6, ST_NONFINITE = 7 };

__device__ __forceinline__ double* red_partials(const Scratch& sc, int slot, int load) {
  return sc.partials + ((long long)slot * kMaxRhs + load) * sc.max_blocks;
}
__device__ __forceinline__ unsigned* red_counter(const Scratch& sc, int slot, int load) {
  return sc.counters + slot * kMaxRhs + load;
}

// ------------------------------------------------------------------------------ scalar logic
// F1 last CTA: stopping test of Alg 2 l.3 with the relative reading.
static __device__ void scalar_after_rnorm(LoadState* st, double rn, double* hist, int hist_stride, int load) {
  st->rn = rn;
  if (!isfinite(rn)) {
    st->status = ST_NONFINITE;
    st->active = 0;
    return;
  }
  const int it = st->iters;
  if (it == 0) {
    st->r0 = rn;
    st->tol_abs = st->rel_tol * rn;
    if (rn <= st->zero_floor) {  // all-zero RHS up to assembly round-off
      st->active = 0;
      st->converged = 1;
    } else if (st->fixed_iters <= 0 && st->max_iter <= 0) {
      st->active = 0;
    }
  } else if (st->fixed_iters > 0) {
    if (it >= st->fixed_iters) {
      st->active = 0;
      st->converged = rn <= st->tol_abs;
    }
  } else {
    if (rn <= st->tol_abs) {
      st->active = 0;
      st->converged = 1;
    } else if (it >= st->max_iter) {
      st->active = 0;
    }
  }
  if (hist && it < hist_stride) hist[(long long)load * hist_stride + it] = st->r0 > 0 ? rn / st->r0 : 0.0;
}

// Per-iteration coefficient record of the solve (hist planes: 0 ||r||_inf / ||r0||_inf, 1 gamma_1,
// 2 alpha; [plane][kMaxRhs][hist_stride]) — the PCG-Lanczos tridiagonal of uno_cg_spectrum.
__device__ __forceinline__ void record_coef(double* hist, int hist_stride, int plane, int load, int it, double v) {
  if (hist && it < hist_stride) hist[((long long)plane * kMaxRhs + load) * hist_stride + it] = v;
}

// G-pass last CTA: gamma_0 <- gamma_1 ; gamma_1 <- r.s ; beta = gamma_1 / gamma_0 (Alg 2 l.7-8).
static __device__ void scalar_after_gamma(LoadState* st, double g1, double* hist = nullptr, int hist_stride = 0,
                                          int load = 0) {
  if (!isfinite(g1)) {
    st->status = ST_NONFINITE;
    st->active = 0;
    return;
  }
  if (!(g1 > 0.0)) {
    st->status = ST_BREAKDOWN;
    st->active = 0;
    return;
  }
  const double g0 = st->iters == 0 ? 1.0 : st->gamma1;
  st->gamma0 = g0;
  st->gamma1 = g1;
  st->beta = st->iters == 0 ? 0.0 : g1 / g0;
  record_coef(hist, hist_stride, 1, load, st->iters, g1);
}

// K last CTA: alpha = gamma_1 / (d.p) (Alg 2 l.10).
static __device__ void scalar_after_dp(LoadState* st, double dp, double* hist = nullptr, int hist_stride = 0,
                                       int load = 0) {
  st->dp = dp;
  if (!isfinite(dp)) {
    st->status = ST_NONFINITE;
    st->active = 0;
    st->pending_u = 0;
    return;
  }
  if (!(dp > 0.0)) {
    st->status = ST_BREAKDOWN;
    st->active = 0;
    st->pending_u = 0;
    return;
  }
  st->alpha_prev = st->alpha;
  st->alpha = st->gamma1 / dp;
  record_coef(hist, hist_stride, 2, load, st->iters, st->alpha);
  st->iters += 1;
  st->pending_u = 1;
}

// ============================================================================== async copy helpers
__device__ __forceinline__ void cp_async16(void* smem_ptr, const void* gptr) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_ptr, const void* gptr) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ============================================================================== G multiply
// s_hat(k) = G_hat(k) r_hat(k) on one bin; returns w_k Re(r_hat^H G_hat r_hat) (Parseval term).
// gtab holds the unique entries in Eq B7 order: v1=G11 v2=G22 v3=G12 v4=G33 v5=G23 v6=G13.
template <int NC>
__device__ __forceinline__ double gmul_bin(double2* const* tiles, int ti, const double* gtab, long long nspec,
                                           long long b, double w) {
  if (NC == 1) {
    const double gv = gtab[b];
    double2 X = tiles[0][ti];
    const double q = w * gv * fma(X.x, X.x, X.y * X.y);
    tiles[0][ti] = make_double2(gv * X.x, gv * X.y);
    return q;
  } else if (NC == 2) {
    const double v1 = gtab[b], v2 = gtab[nspec + b], v3 = gtab[2 * nspec + b];
    const double2 X1 = tiles[0][ti], X2 = tiles[1][ti];
    const double2 Y1 = make_double2(fma(v1, X1.x, v3 * X2.x), fma(v1, X1.y, v3 * X2.y));
    const double2 Y2 = make_double2(fma(v3, X1.x, v2 * X2.x), fma(v3, X1.y, v2 * X2.y));
    tiles[0][ti] = Y1;
    tiles[1][ti] = Y2;
    return w * (X1.x * Y1.x + X1.y * Y1.y + X2.x * Y2.x + X2.y * Y2.y);
  } else {
    const double v1 = gtab[b], v2 = gtab[nspec + b], v3 = gtab[2 * nspec + b];
    const double v4 = gtab[3 * nspec + b], v5 = gtab[4 * nspec + b], v6 = gtab[5 * nspec + b];
    const double2 X1 = tiles[0][ti], X2 = tiles[1][ti], X3 = tiles[2][ti];
    double2 Y1, Y2, Y3;
    Y1.x = fma(v1, X1.x, fma(v3, X2.x, v6 * X3.x));
    Y1.y = fma(v1, X1.y, fma(v3, X2.y, v6 * X3.y));
    Y2.x = fma(v3, X1.x, fma(v2, X2.x, v5 * X3.x));
    Y2.y = fma(v3, X1.y, fma(v2, X2.y, v5 * X3.y));
    Y3.x = fma(v6, X1.x, fma(v5, X2.x, v4 * X3.x));
    Y3.y = fma(v6, X1.y, fma(v5, X2.y, v4 * X3.y));
    tiles[0][ti] = Y1;
    tiles[1][ti] = Y2;
    tiles[2][ti] = Y3;
    return w * (X1.x * Y1.x + X1.y * Y1.y + X2.x * Y2.x + X2.y * Y2.y + X3.x * Y3.x + X3.y * Y3.y);
  }
}

// Same multiply on NC register values of one bin (fused-butterfly variant).
template <int NC>
__device__ __forceinline__ double gmul_vals(double2* x, const double* gtab, long long nspec, long long b, double w) {
  if (NC == 1) {
    const double gv = gtab[b];
    const double q = w * gv * fma(x[0].x, x[0].x, x[0].y * x[0].y);
    x[0] = make_double2(gv * x[0].x, gv * x[0].y);
    return q;
  } else if (NC == 2) {
    const double v1 = gtab[b], v2 = gtab[nspec + b], v3 = gtab[2 * nspec + b];
    const double2 X1 = x[0], X2 = x[1];
    const double2 Y1 = make_double2(fma(v1, X1.x, v3 * X2.x), fma(v1, X1.y, v3 * X2.y));
    const double2 Y2 = make_double2(fma(v3, X1.x, v2 * X2.x), fma(v3, X1.y, v2 * X2.y));
    x[0] = Y1;
    x[1] = Y2;
    return w * (X1.x * Y1.x + X1.y * Y1.y + X2.x * Y2.x + X2.y * Y2.y);
  } else {
    const double v1 = gtab[b], v2 = gtab[nspec + b], v3 = gtab[2 * nspec + b];
    const double v4 = gtab[3 * nspec + b], v5 = gtab[4 * nspec + b], v6 = gtab[5 * nspec + b];
    const double2 X1 = x[0], X2 = x[1], X3 = x[2];
    double2 Y1, Y2, Y3;
    Y1.x = fma(v1, X1.x, fma(v3, X2.x, v6 * X3.x));
    Y1.y = fma(v1, X1.y, fma(v3, X2.y, v6 * X3.y));
    Y2.x = fma(v3, X1.x, fma(v2, X2.x, v5 * X3.x));
    Y2.y = fma(v3, X1.y, fma(v2, X2.y, v5 * X3.y));
    Y3.x = fma(v6, X1.x, fma(v5, X2.x, v4 * X3.x));
    Y3.y = fma(v6, X1.y, fma(v5, X2.y, v4 * X3.y));
    x[0] = Y1;
    x[1] = Y2;
    x[2] = Y3;
    return w * (X1.x * Y1.x + X1.y * Y1.y + X2.x * Y2.x + X2.y * Y2.y + X3.x * Y3.x + X3.y * Y3.y);
  }
}

__device__ __forceinline__ double parseval_w(int kx, int M) { return (kx == 0 || kx == M) ? 1.0 : 2.0; }

// Per-CTA partial of a reduction: deterministic block reduce, thread 0 stores the partial.
// The fixed-order combine over CTAs and the CG scalar logic run in scalar_kernel (a 1-CTA-per-
// load launch right after the producing pass) so no CTA waits on a global atomic at its end.
template <bool MAX>
__device__ __forceinline__ void partial_write(const Ctx& cx, int slot, int load, int my, double v, double* red_sh) {
  const double b = block_reduce<MAX>(v, red_sh);
  if (threadIdx.x == 0) red_partials(cx.sc, slot, load)[my] = b;
}

static __device__ void gamma_finish(const Ctx& cx, int load, double part, double* red_sh, int mode) {
  (void)mode;
  partial_write<false>(cx, RED_GAMMA, load, blockIdx.x, part, red_sh);
}

static __device__ void dp_finish(const Ctx& cx, int load, int nblk, int my, double part, double* red_sh, int mode) {
  (void)nblk;
  (void)mode;
  partial_write<false>(cx, RED_DP, load, my, part, red_sh);
}

}  // namespace uno
