// elastic_modal.cuh — exact Q1 hexahedral elasticity element in the Walsh-Hadamard modal basis,
// computed at compile time in integer arithmetic (independent of oracle/, which integrates by
// Gauss quadrature in floating point).
//
// Unit cube, shape functions N_a = prod_t phi_{a_t}(x_t), phi_0 = 1 - x, phi_1 = x, corner
// a = a_x + 2 a_y + 4 a_z, dof (a, alpha) -> 3a + alpha.  With the exact 1D integrals
//   int phi_a phi_b = (a == b ? 2 : 1)/6,   int phi_a' phi_b' = (a == b ? 1 : -1),
//   int phi_a' phi_b = (a ? 1 : -1)/2,
// every entry of K_lam = int (dN_a/dx_alpha)(dN_b/dx_beta) and
// K_mu = delta_ab sum_j int dN_a/dx_j dN_b/dx_j + int (dN_a/dx_beta)(dN_b/dx_alpha)
// (D = lam I(x)I + 2 mu I^s, Eq 80) is an integer multiple of 1/72; an element of edge
// h scales by h.  The Hadamard transform H[m][a] = (-1)^popcount(m & a) block-diagonalises
// them (45 nonzeros of 576): K_e u = H K^ H u with
//   K^ = (h / (72 * 64)) (lam KLH + mu KMH),  KLH = H KL H,  KMH = H KM H  (integers).
#pragma once

#include <utility>

namespace uno {
namespace modal {

struct IMat24 {
  long long v[24][24];
};

__host__ __device__ constexpr int popc3(int x) { return (x & 1) + ((x >> 1) & 1) + ((x >> 2) & 1); }

// int over the unit cube of d_i N_a * d_j N_b, times 72
__host__ __device__ constexpr long long grad_int72(int i, int j, int a, int b) {
  long long num = 1, den = 1;
  for (int t = 0; t < 3; ++t) {
    const int at = (a >> t) & 1, bt = (b >> t) & 1;
    if (t == i && t == j) {
      num *= (at == bt ? 1 : -1);
    } else if (t == i) {
      num *= (at ? 1 : -1);
      den *= 2;
    } else if (t == j) {
      num *= (bt ? 1 : -1);
      den *= 2;
    } else {
      num *= (at == bt ? 2 : 1);
      den *= 6;
    }
  }
  return num * 72 / den;
}

__host__ __device__ constexpr IMat24 make_KL() {
  IMat24 K{};
  for (int a = 0; a < 8; ++a)
    for (int al = 0; al < 3; ++al)
      for (int b = 0; b < 8; ++b)
        for (int be = 0; be < 3; ++be) K.v[3 * a + al][3 * b + be] = grad_int72(al, be, a, b);
  return K;
}

__host__ __device__ constexpr IMat24 make_KM() {
  IMat24 K{};
  for (int a = 0; a < 8; ++a)
    for (int al = 0; al < 3; ++al)
      for (int b = 0; b < 8; ++b)
        for (int be = 0; be < 3; ++be) {
          long long s = grad_int72(be, al, a, b);
          if (al == be)
            for (int j = 0; j < 3; ++j) s += grad_int72(j, j, a, b);
          K.v[3 * a + al][3 * b + be] = s;
        }
  return K;
}

__host__ __device__ constexpr IMat24 hadamard(const IMat24& K) {
  IMat24 T{}, R{};
  for (int m = 0; m < 8; ++m)
    for (int al = 0; al < 3; ++al)
      for (int c = 0; c < 24; ++c) {
        long long s = 0;
        for (int a = 0; a < 8; ++a) s += ((popc3(m & a) & 1) ? -1 : 1) * K.v[3 * a + al][c];
        T.v[3 * m + al][c] = s;
      }
  for (int r = 0; r < 24; ++r)
    for (int n = 0; n < 8; ++n)
      for (int be = 0; be < 3; ++be) {
        long long s = 0;
        for (int b = 0; b < 8; ++b) s += ((popc3(n & b) & 1) ? -1 : 1) * T.v[r][3 * b + be];
        R.v[r][3 * n + be] = s;
      }
  return R;
}

constexpr IMat24 KLH = hadamard(make_KL());
constexpr IMat24 KMH = hadamard(make_KM());

__host__ __device__ constexpr long long klh(int r, int c) { return KLH.v[r][c]; }
__host__ __device__ constexpr long long kmh(int r, int c) { return KMH.v[r][c]; }

constexpr int count_nz() {
  int n = 0;
  for (int r = 0; r < 24; ++r)
    for (int c = 0; c < 24; ++c) n += (KLH.v[r][c] != 0 || KMH.v[r][c] != 0);
  return n;
}
static_assert(count_nz() == 45, "Walsh-Hadamard modal Q1 elasticity operator has 45 nonzeros");

// v_hat[r] += (ls * KLH[r][c] + ms * KMH[r][c]) * u_hat[c] over the nonzeros, unrolled at
// compile time by a fold over the 576 (r, c) positions (integer entries become immediates).
template <int R, int C>
__device__ __forceinline__ void modal_term(double* vh, const double* uh, double ls, double ms) {
  if constexpr (klh(R, C) != 0 || kmh(R, C) != 0) {
    double coef;
    if constexpr (klh(R, C) != 0 && kmh(R, C) != 0)
      coef = fma(ls, (double)klh(R, C), ms * (double)kmh(R, C));
    else if constexpr (klh(R, C) != 0)
      coef = ls * (double)klh(R, C);
    else
      coef = ms * (double)kmh(R, C);
    vh[R] = fma(coef, uh[C], vh[R]);
  }
}

template <int R0, int... I>
__device__ __forceinline__ void modal_apply_seq(double* vh, const double* uh, double ls, double ms,
                                                std::integer_sequence<int, I...>) {
  (modal_term<R0 + I / 24, I % 24>(vh, uh, ls, ms), ...);
}

// rows R0 .. 23 (rows of a zero mode may be skipped by the caller)
template <int R0>
__device__ __forceinline__ void modal_apply(double* vh, const double* uh, double ls, double ms) {
  modal_apply_seq<R0>(vh, uh, ls, ms, std::make_integer_sequence<int, (24 - R0) * 24>{});
}

// The 45 nonzeros form small blocks with repeated entries (rows/cols = 3 * mode + component):
//   A = {3, 7, 14}        288 lam J + 576 mu I        (J = all-ones block)
//   {4, 6} {5, 12} {8, 13} 288 mu J
//   {9, 20} {10, 17} {15, 19}  96 lam J + 288 mu I
//   E = {11, 16, 18}       96 mu (J + I)
//   F = {21}, {22}, {23}   32 lam + 128 mu
//   rows / cols 0, 1, 2 (mode 0, the rigid translations) zero.
// apply_blocked evaluates K^ u in that form: 40 DP operations instead of 45 FMAs plus the
// per-entry coefficients.  blocked_matches() re-derives both integer matrices from this
// description and the static_assert pins it to KLH / KMH.
struct BlockDesc {
  long long L[24][24], M[24][24];
};
__host__ __device__ constexpr BlockDesc blocked_desc() {
  BlockDesc B{};
  const int A[3] = {3, 7, 14};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      B.L[A[i]][A[j]] = 288;
      B.M[A[i]][A[j]] = i == j ? 576 : 0;
    }
  const int P[3][2] = {{4, 6}, {5, 12}, {8, 13}};
  const int D[3][2] = {{9, 20}, {10, 17}, {15, 19}};
  for (int q = 0; q < 3; ++q)
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        B.M[P[q][i]][P[q][j]] = 288;
        B.L[D[q][i]][D[q][j]] = 96;
        B.M[D[q][i]][D[q][j]] = i == j ? 288 : 0;
      }
  const int E[3] = {11, 16, 18};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) B.M[E[i]][E[j]] = i == j ? 192 : 96;
  for (int r = 21; r < 24; ++r) {
    B.L[r][r] = 32;
    B.M[r][r] = 128;
  }
  return B;
}
__host__ __device__ constexpr bool blocked_matches() {
  const BlockDesc B = blocked_desc();
  for (int r = 0; r < 24; ++r)
    for (int c = 0; c < 24; ++c)
      if (B.L[r][c] != KLH.v[r][c] || B.M[r][c] != KMH.v[r][c]) return false;
  return true;
}
static_assert(blocked_matches(), "block form of the modal Q1 elasticity operator");

// v[3..23] = (ls KLH + ms KMH) u (ls, ms already scaled by h / (72 * 64)); v[0..2] = 0
__device__ __forceinline__ void apply_blocked(double* v, const double* u, double ls, double ms) {
  const double l288 = 288.0 * ls, m576 = 576.0 * ms, m288 = 288.0 * ms, l96 = 96.0 * ls, m96 = 96.0 * ms;
  v[0] = v[1] = v[2] = 0.0;
  {
    const double t = l288 * (u[3] + u[7] + u[14]);
    v[3] = fma(m576, u[3], t);
    v[7] = fma(m576, u[7], t);
    v[14] = fma(m576, u[14], t);
  }
  v[4] = v[6] = m288 * (u[4] + u[6]);
  v[5] = v[12] = m288 * (u[5] + u[12]);
  v[8] = v[13] = m288 * (u[8] + u[13]);
  {
    const double t9 = l96 * (u[9] + u[20]), t10 = l96 * (u[10] + u[17]), t15 = l96 * (u[15] + u[19]);
    v[9] = fma(m288, u[9], t9);
    v[20] = fma(m288, u[20], t9);
    v[10] = fma(m288, u[10], t10);
    v[17] = fma(m288, u[17], t10);
    v[15] = fma(m288, u[15], t15);
    v[19] = fma(m288, u[19], t15);
  }
  {
    const double t = m96 * (u[11] + u[16] + u[18]);
    v[11] = fma(m96, u[11], t);
    v[16] = fma(m96, u[16], t);
    v[18] = fma(m96, u[18], t);
  }
  const double f = fma(32.0, ls, 128.0 * ms);
  v[21] = f * u[21];
  v[22] = f * u[22];
  v[23] = f * u[23];
}

// In-place 8-point Walsh-Hadamard transform over corners (natural order, unnormalised).
__device__ __forceinline__ void wht8(double* v /* stride 3 */) {
#pragma unroll
  for (int b = 1; b < 8; b <<= 1)
#pragma unroll
    for (int a = 0; a < 8; ++a)
      if (!(a & b)) {
        const double x = v[3 * a], y = v[3 * (a | b)];
        v[3 * a] = x + y;
        v[3 * (a | b)] = x - y;
      }
}

// The x and y stages of wht8 on the 4 corners of one node plane (stride 3).
__device__ __forceinline__ void wht4(double* v) {
#pragma unroll
  for (int b = 1; b < 4; b <<= 1)
#pragma unroll
    for (int a = 0; a < 4; ++a)
      if (!(a & b)) {
        const double x = v[3 * a], y = v[3 * (a | b)];
        v[3 * a] = x + y;
        v[3 * (a | b)] = x - y;
      }
}

}  // namespace modal
}  // namespace uno
