// fft.cuh — fp64 complex FFT of 8 interleaved sequences held in shared memory (Stockham
// autosort, radix 4/8/16 butterflies in registers).  Used by every transform pass of the
// UNO apply T^H Q T (Eq 47-48; cost model Eq 54).  Unnormalised: forward uses
// e^{-2 pi i jk/L}, inverse e^{+2 pi i jk/L}; the 1/n of the unitary pair is folded into
// the tabulated symbol.
//
// Shared-memory tile: element j (0..L-1) of column c (0..7) lives at
//     idx(j, c) = 8*j + (c ^ (j & 7))
// The XOR swizzle makes both the column-contiguous accesses of the butterflies and the
// row-contiguous (transposing) global<->smem copies bank-conflict free for 16-byte
// double2 elements.
#pragma once
#include "common.cuh"

namespace uno {

__device__ __forceinline__ int tidx(int j, int c) { return (j << 3) + (c ^ (j & 7)); }

constexpr double kR2 = 0.70710678118654752440;   // cos(pi/4)
constexpr double kC8 = 0.92387953251128675613;   // cos(pi/8)
constexpr double kS8 = 0.38268343236508977173;   // sin(pi/8)

template <int R> struct Dft;

template <> struct Dft<2> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <> struct Dft<4> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    double2 a2 = cadd(v[1], v[3]), a3 = csub(v[1], v[3]);
    v[0] = cadd(a0, a2);
    v[2] = csub(a0, a2);
    v[1] = cadd(a1, mul_mi(a3));
    v[3] = csub(a1, mul_mi(a3));
  }
};

// w8^1 * o, w8^3 * o with w8 = e^{-i pi/4}
__device__ __forceinline__ double2 mul_w8_1(double2 o) { return make_double2((o.x + o.y) * kR2, (o.y - o.x) * kR2); }
__device__ __forceinline__ double2 mul_w8_3(double2 o) { return make_double2((o.y - o.x) * kR2, -(o.x + o.y) * kR2); }

template <> struct Dft<8> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4>::run(e);
    Dft<4>::run(o);
    double2 t1 = mul_w8_1(o[1]), t2 = mul_mi(o[2]), t3 = mul_w8_3(o[3]);
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], t1);
    v[5] = csub(e[1], t1);
    v[2] = cadd(e[2], t2);
    v[6] = csub(e[2], t2);
    v[3] = cadd(e[3], t3);
    v[7] = csub(e[3], t3);
  }
};

template <> struct Dft<16> {
  // 4 x 4: X[k1 + 4 k2] = sum_{n2} w16^{n2 k1} w4^{n2 k2} sum_{n1} v[4 n1 + n2] w4^{n1 k1}
  static __device__ __forceinline__ void run(double2* v) {
    double2 a[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      double2 t[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
      Dft<4>::run(t);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) a[n2][k1] = t[k1];
    }
    // twiddles w16^{n2 k1}
    const double2 w1 = make_double2(kC8, -kS8), w3 = make_double2(kS8, -kC8), w9 = make_double2(-kC8, kS8);
    a[1][1] = cmul(a[1][1], w1);
    a[1][2] = mul_w8_1(a[1][2]);
    a[1][3] = cmul(a[1][3], w3);
    a[2][1] = mul_w8_1(a[2][1]);
    a[2][2] = mul_mi(a[2][2]);
    a[2][3] = mul_w8_3(a[2][3]);
    a[3][1] = cmul(a[3][1], w3);
    a[3][2] = mul_w8_3(a[3][2]);
    a[3][3] = cmul(a[3][3], w9);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 t[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
      Dft<4>::run(t);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[k2];
    }
  }
};

__host__ __device__ constexpr int pick_radix(int rem) {
  return (rem == 32 || rem == 64 || rem == 512) ? 8 : (rem >= 16 ? 16 : rem);
}
__host__ __device__ constexpr int min_radix(int L, int ns = 1) {
  return ns >= L ? 1 << 30
                 : (pick_radix(L / ns) < min_radix(L, ns * pick_radix(L / ns)) ? pick_radix(L / ns)
                                                                                : min_radix(L, ns * pick_radix(L / ns)));
}
// threads needed so that every Stockham stage has one butterfly per thread
__host__ __device__ constexpr int fft_threads(int L) { return (8 * L / min_radix(L)) < 64 ? 64 : 8 * L / min_radix(L); }

// One Stockham stage (radix R, span NS) over the 8 columns of the tile, in place.
template <int L, int R, int NS, bool INV>
__device__ __forceinline__ void fft_stage(double2* s, const double2* __restrict__ tw) {
  constexpr int NJ = L / R;
  constexpr int ITEMS = NJ * kTile;
  const int t = threadIdx.x;
  const bool act = t < ITEMS;
  const int c = t & 7, j = t >> 3;
  const int k = j % NS;
  double2 v[R];
  if (act) {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[tidx(j + r * NJ, c)];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = tw[r * k * (L / (NS * R))];
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    if (INV) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
    }
    Dft<R>::run(v);
    if (INV) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
    }
  }
  __syncthreads();
  if (act) {
    const int base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) s[tidx(base + r * NS, c)] = v[r];
  }
  __syncthreads();
}

// ---- the same Stockham stages on a tile of W (power of two <= 8) columns: idx_w(j, c) =
// W j + (c ^ (j & (W-1))).  Narrow tiles let a long transform (L = 1024) keep two CTAs per SM.
template <int W>
__device__ __forceinline__ int tidx_w(int j, int c) { return j * W + (c ^ (j & (W - 1))); }

// TT: threads of the CTA when fewer than one per butterfly (0: one butterfly per thread, inactive
// threads allowed).  With TT > 0 a thread runs ITEMS / TT butterflies of the stage, which is how a
// radix-16 plan stays under its register budget without spills (1024-point DST: 256 threads at
// 128 registers instead of 512 at 64).
template <int L, int R, int NS, bool INV, int W, int TT = 0>
__device__ __forceinline__ void fft_stage_w(double2* s, const double2* __restrict__ tw) {
  constexpr int NJ = L / R;
  constexpr int ITEMS = NJ * W;
  constexpr int NH = TT > 0 ? ITEMS / TT : 1;
  static_assert(TT == 0 || (ITEMS % TT == 0 && TT % W == 0), "whole butterflies per thread");
  const int t = threadIdx.x;
  const bool act = TT > 0 || t < ITEMS;
  const int c = t & (W - 1), j0 = t / W;
  double2 v[NH][R];
  if (act) {
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int j = j0 + h * (TT > 0 ? TT / W : 0), k = j % NS;
#pragma unroll
      for (int r = 0; r < R; ++r) v[h][r] = s[tidx_w<W>(j + r * NJ, c)];
      if (NS > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = tw[r * k * (L / (NS * R))];
          if (INV) w.y = -w.y;
          v[h][r] = cmul(v[h][r], w);
        }
      }
      if (INV) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[h][r].y = -v[h][r].y;
      }
      Dft<R>::run(v[h]);
      if (INV) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[h][r].y = -v[h][r].y;
      }
    }
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int j = j0 + h * (TT > 0 ? TT / W : 0), k = j % NS, base = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) s[tidx_w<W>(base + r * NS, c)] = v[h][r];
    }
  }
  __syncthreads();
}
template <int L, int NS, bool INV, int W, int TT = 0>
struct FftStagesW {
  static __device__ __forceinline__ void run(double2* s, const double2* tw) {
    constexpr int R = pick_radix(L / NS);
    fft_stage_w<L, R, NS, INV, W, TT>(s, tw);
    FftStagesW<L, NS * R, INV, W, TT>::run(s, tw);
  }
};
template <int L, bool INV, int W, int TT>
struct FftStagesW<L, L, INV, W, TT> {
  static __device__ __forceinline__ void run(double2*, const double2*) {}
};

template <int L, int NS, bool INV>
struct FftStages {
  static __device__ __forceinline__ void run(double2* s, const double2* tw) {
    constexpr int R = pick_radix(L / NS);
    fft_stage<L, R, NS, INV>(s, tw);
    FftStages<L, NS * R, INV>::run(s, tw);
  }
};
template <int L, bool INV>
struct FftStages<L, L, INV> {
  static __device__ __forceinline__ void run(double2*, const double2*) {}
};

// Full length-L transform of the 8 tile columns.  Caller syncs before (data in smem).
template <int L, bool INV>
__device__ __forceinline__ void fft_tile(double2* s, const double2* tw) {
  FftStages<L, 1, INV>::run(s, tw);
}

template <int L, bool INV, int W, int TT = 0>
__device__ __forceinline__ void fft_tile_w(double2* s, const double2* tw) {
  FftStagesW<L, 1, INV, W, TT>::run(s, tw);
}
__host__ __device__ constexpr int fft_threads_w(int L, int W) {
  return (W * L / min_radix(L)) < 64 ? 64 : W * L / min_radix(L);
}

// ---- NT tiles at once (tile q at s + q*8L): more butterflies per stage for bigger CTAs ----
// ALL: the CTA has exactly ITEMS threads (no inactive thread).  Inside a loop over tiles the
// `if (act)` form would keep v[] live around the loop (undefined on the inactive path = the
// previous iteration's value), i.e. R complex registers pinned through every other stage.
template <int L, int NT, int R, int NS, bool INV, bool ALL = false>
__device__ __forceinline__ void fft_stage_nt(double2* s, const double2* __restrict__ tw) {
  constexpr int NJ = L / R;
  constexpr int ITEMS = NJ * kTile * NT;
  const int t = threadIdx.x;
  const bool act = ALL || t < ITEMS;
  const int q = t / (NJ * kTile), rem = t - q * (NJ * kTile);
  const int c = rem & 7, j = rem >> 3;
  const int k = j % NS;
  double2* sq = s + q * 8 * L;
  double2 v[R];
  if (act) {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = sq[tidx(j + r * NJ, c)];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = tw[r * k * (L / (NS * R))];
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    if (INV) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
    }
    Dft<R>::run(v);
    if (INV) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
    }
  }
  __syncthreads();
  if (act) {
    const int base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) sq[tidx(base + r * NS, c)] = v[r];
  }
  __syncthreads();
}

template <int L, int NT, int NS, bool INV, bool ALL = false>
struct FftStagesNT {
  static __device__ __forceinline__ void run(double2* s, const double2* tw) {
    constexpr int R = pick_radix(L / NS);
    fft_stage_nt<L, NT, R, NS, INV, ALL>(s, tw);
    FftStagesNT<L, NT, NS * R, INV, ALL>::run(s, tw);
  }
};
template <int L, int NT, bool INV, bool ALL>
struct FftStagesNT<L, NT, L, INV, ALL> {
  static __device__ __forceinline__ void run(double2*, const double2*) {}
};

template <int R>
__device__ __forceinline__ void dft_reg_inv_inline(double2* v) {
#pragma unroll
  for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
  Dft<R>::run(v);
#pragma unroll
  for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
}

template <int L, int NT, bool INV>
__device__ __forceinline__ void fft_tiles(double2* s, const double2* tw) {
  FftStagesNT<L, NT, 1, INV>::run(s, tw);
}
// threads for one butterfly per thread in every stage of NT tiles
__host__ __device__ constexpr int fft_threads_nt(int L, int NT) {
  return (NT * 8 * L / min_radix(L)) < 64 ? 64 : NT * 8 * L / min_radix(L);
}

// ---- forward FFT -> per-bin operator -> inverse FFT, with the operator fused into the middle
// butterfly: the last forward stage (radix R, span L/R) produces, per thread, the R bins
// j + r L/R in registers; they are exactly the inputs of the first inverse stage (radix R,
// span 1) when the plan's first and last radices agree, so the symbol multiply needs no extra
// shared-memory round trip or barrier.
__host__ __device__ constexpr int plan_ns(int L, int s) {  // span of stage s
  return s == 0 ? 1 : plan_ns(L, s - 1) * pick_radix(L / plan_ns(L, s - 1));
}
__host__ __device__ constexpr int plan_stages(int L, int ns = 1) {
  return ns >= L ? 0 : 1 + plan_stages(L, ns * pick_radix(L / ns));
}
__host__ __device__ constexpr int plan_radix(int L, int s) { return pick_radix(L / plan_ns(L, s)); }
__host__ __device__ constexpr bool gconv_fusable(int L) {
  return plan_stages(L) >= 2 && plan_radix(L, 0) == plan_radix(L, plan_stages(L) - 1);
}

template <int L, int NT, int NS, int STOP, bool INV, bool ALL = false>
struct FftStagesNTUntil {
  static __device__ __forceinline__ void run(double2* s, const double2* tw) {
    if constexpr (NS < STOP) {
      constexpr int R = pick_radix(L / NS);
      fft_stage_nt<L, NT, R, NS, INV, ALL>(s, tw);
      FftStagesNTUntil<L, NT, NS * R, STOP, INV, ALL>::run(s, tw);
    }
  }
};

// op(int tile, int col, int kbin, double2* x /*NC values of that bin*/) -> Parseval term;
// modifies x in place.  Returns the thread's sum of op results.  Caller syncs before.
struct GconvNoHook {
  __device__ __forceinline__ void operator()(int) const {}
};
// pre(q): called before component q's forward stages (e.g. wait for its copy group + barrier);
// post(q): after its inverse stages (the tile is complete: e.g. store it while the next one runs).
template <int L, int NT, int NC, bool ALL = false, class Op, class Pre = GconvNoHook, class Post = GconvNoHook>
__device__ __forceinline__ double fft_gconv(double2* const* tiles, const double2* __restrict__ tw, Op op,
                                            Pre pre = Pre(), Post post = Post()) {
  constexpr int S = plan_stages(L);
  constexpr int RL = plan_radix(L, S - 1);
  constexpr int NJ = L / RL;
  static_assert(gconv_fusable(L), "first and last radix must agree");
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    pre(q);
    FftStagesNTUntil<L, NT, 1, NJ, false, ALL>::run(tiles[q], tw);
  }
  constexpr int ITEMS = NJ * kTile * NT;
  const int t = threadIdx.x;
  const bool act = ALL || t < ITEMS;
  const int tq = t / (NJ * kTile), rem = t - tq * (NJ * kTile);
  const int c = rem & 7, j = rem >> 3;
  double part = 0.0;
  double2 v[NC][RL];
  if (act) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const double2* sq = tiles[q] + tq * 8 * L;
#pragma unroll
      for (int r = 0; r < RL; ++r) v[q][r] = sq[tidx(j + r * NJ, c)];
#pragma unroll
      for (int r = 1; r < RL; ++r) v[q][r] = cmul(v[q][r], tw[r * j]);  // last-stage twiddles (span NJ)
      Dft<RL>::run(v[q]);
    }
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      double2 x[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) x[q] = v[q][r];
      part += op(tq, c, j + r * NJ, x);
#pragma unroll
      for (int q = 0; q < NC; ++q) v[q][r] = x[q];
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) dft_reg_inv_inline<RL>(v[q]);  // first inverse stage (span 1)
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double2* sq = tiles[q] + tq * 8 * L;
#pragma unroll
      for (int r = 0; r < RL; ++r) sq[tidx(j * RL + r, c)] = v[q][r];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    FftStagesNT<L, NT, plan_radix(L, 0), true, ALL>::run(tiles[q], tw);
    post(q);
  }
  return part;
}

// In-register forward/inverse DFT of length R (R = 2, 4, 8, 16).
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(double2* v) {
  if (INV) {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
  }
  Dft<R>::run(v);
  if (INV) {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r].y = -v[r].y;
  }
}

// Half of an NB-point DFT: the outputs k = 2m + h (m < NB/2) of X[k] = sum_r v_r w^{rk}
// (w = w_NB, conjugated for INV) as an NB/2-point DFT of v_r + v_{r+NB/2} (h = 0) or of
// (v_r - v_{r+NB/2}) w^r (h = 1).  Two threads per sequence keep every thread of the CTA busy
// in the across-row DFT of F1/F3 (H1 = M + 1 sequences only) and in
// the x pass (8 rows x 8 sequences of 16).  twb[r] = w_NB^r, r < NB/2.
template <int NB, bool INV>
__device__ __forceinline__ void dft_half(const double2* v, int h, const double2* twb, double2* o) {
  constexpr int NH = NB / 2;
#pragma unroll
  for (int r = 0; r < NH; ++r) {
    const double2 a = v[r], b = v[r + NH];
    o[r] = h == 0 ? cadd(a, b) : cmul(csub(a, b), INV ? cconj(twb[r]) : twb[r]);
  }
  dft_reg<NH, INV>(o);
}

}  // namespace uno
