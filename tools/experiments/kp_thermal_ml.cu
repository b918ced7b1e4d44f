// EXPERIMENT (not built into libunocg.so): multi-load thermal K, measured slower than the
// production kp_thermal3d_rn_kernel<4> on B200 (256^3 x 3 loads: 242 us L=3 / 315 us L=2 /
// 263 us L=1 at 16 warps vs 202 us; ncu L=3: 8 warps/SM, issue 38 %, stalls wait/selected/short
// scoreboard).  Kept for reference; see DESIGN.md §5 "Measured and rejected".
// kp_thermal.cu — matrix-free Q1 heat-conduction K.d with the fused d.p partial (Alg 2
// l.9-10, Eq 22 with the element of App. A1 / SURVEY A1) for several load cases per CTA.
//
// Q1 element (unit kappa, cube of edge h): K_e = kappa h {1/3 diag, 0 edge, -1/12 face / body
// diagonal}.  Gathered at node i over its 8 elements e (S_e = sum of the element's 8 corner
// values, W_j = sum of kappa over the 4 elements sharing the edge i-j):
//   p_i = h/12 [ 5 d_i sum_e kappa_e + sum_{6 axis nbrs j} W_j d_j - sum_e kappa_e S_e ].
// Everything that depends on the phase field only (kappa selects, the 8-element and edge sums)
// is identical for every load case, so one thread computes its NR = 2 node rows for all L load
// cases of its CTA and pays for the kappa work once (ncu of the one-load kernel: ~18 of its 72
// instructions per node were kappa work, 10 of them the byte->kappa selects).  Box sums S_e are
// separable (x pairs -> (x,y) quads -> two planes) and shared between the thread's two rows and
// between consecutive planes of the z march; the tile is 32 x 16 nodes x ZC planes, 256 threads.
// d planes of the L loads and the phase layer stream through an 8-slot ring with 16-byte
// cp.async four planes ahead.  kappa is pre-scaled by h/12.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dev_common.cuh"
#include "kernels.cuh"

namespace uno {

constexpr int KML_T = 256, KML_TX = 32, KML_TH = 16, KML_NR = 2;
constexpr int KML_DW = 36, KML_DR = KML_TH + 2, KML_DPL = KML_DR * KML_DW;  // d rows y0-1 .. y0+16
constexpr int KML_NCH = KML_DR * (KML_DW / 2);                               // 16-byte chunks / load / plane
constexpr int KML_PW = 64, KML_PR = KML_TH + 1, KML_PHS = KML_PR * KML_PW;   // phase rows y0-1 .. y0+15
constexpr int KML_NPC = KML_PHS / 16;
constexpr int KML_RING = 8, KML_LA = 4;
#ifndef UNO_KML_L
#define UNO_KML_L 3  // load cases per CTA (A/B builds: 1 or 2)
#endif
#ifndef UNO_KML_MINB
#define UNO_KML_MINB 1  // resident CTAs per SM requested from ptxas (2 caps registers at 128)
#endif
constexpr int KML_LMAX = UNO_KML_L;

__host__ __device__ constexpr int kml_smem_bytes(int L) {
  return KML_RING * (L * KML_DPL * (int)sizeof(double) + KML_PHS);
}

template <int L>
struct KMLState {  // carried from the step that read node plane j-1 to the one reading plane j
  double Qk[L][KML_NR + 1][2];  // (x, y) quads of d on plane j-1, per load
  double KSlo[L][KML_NR];       // sum of kappa_e S_e over the 4 elements of layer j-2 at each node
                                // (the lower layer of plane j-1)
  double pp[L][KML_NR];         // partial p of plane j-1: in-plane terms + its z- neighbour
  double cp[L][KML_NR];         // d of plane j-1 at the thread's nodes
  double Klo[KML_NR], Kxlo[KML_NR], Kylo[KML_NR];  // kappa sums of layer j-1 (load independent)
};

// Node plane j arrives; layers j-1 and j (kappa) are resident.  p of plane j-1 is completed with
// plane j's centre value and the box sums of layer j-1; p of plane j is started from its in-plane
// terms.  Carrying only the partial p (instead of plane j-1's in-plane values) keeps the state
// at 12 doubles per load and node pair.
template <int L, bool DZ>
__global__ void __launch_bounds__(KML_T, UNO_KML_MINB) kp_thermal3d_ml_kernel(Ctx cx, int mode, const double* __restrict__ src,
                                                                  double* __restrict__ dst, int ZC) {
  constexpr int T = KML_T, TX = KML_TX, TH = KML_TH, NR = KML_NR;
  constexpr int DW = KML_DW, DPL = KML_DPL, NCH = KML_NCH, PW = KML_PW, PHS = KML_PHS, NPC = KML_NPC;
  constexpr int RING = KML_RING, LA = KML_LA;
  constexpr int NDC = (L * NCH + T - 1) / T;
  static_assert(LA >= 2 && LA < RING, "ring slot of plane k+LA must not be read at step k-1");
  const Geo g = cx.g;
  const int nzc = (g.P3 + ZC - 1) / ZC;
  const int lg = blockIdx.z / nzc;
  const int zcI = blockIdx.z - lg * nzc;
  const int l0 = lg * L;
  unsigned act = 0;
#pragma unroll
  for (int l = 0; l < L; ++l)
    if (l0 + l < g.nrhs && (mode != CG || cx.st[l0 + l].active)) act |= 1u << l;
  if (!act) return;
  extern __shared__ double ksm[];
  double* D = ksm;                                                            // [RING][L][DR][DW]
  unsigned char* PH = reinterpret_cast<unsigned char*>(D + RING * L * DPL);  // [RING][PR][PW]
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int tx = t % TX, ty = t / TX;  // node rows NR ty, NR ty + 1
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TH;
  const int dz = DZ ? 1 : 0;
  const int zs = zcI * ZC + dz;  // first output node plane (full-grid numbering)
  const int ze = min(zs + ZC, g.P3 + dz);
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const long long plane = (long long)N1 * N2;
  const double hc = g.h * (1.0 / 12.0);
  const double k0 = cx.mat[0][0] * hc, k1 = cx.mat[1][0] * hc;
  // staging map: chunk j of this thread -> (load, row, 16-byte column pair)
  long long goffD[NDC];
  unsigned sD[NDC];
  unsigned vD = 0;
#pragma unroll
  for (int m = 0; m < NDC; ++m) {
    const int j = t + m * T;
    const int jj = min(j, L * NCH - 1);
    const int l = jj / NCH, r = jj - l * NCH;
    const int ly = r / (DW / 2), q = r - ly * (DW / 2);
    goffD[m] = (long long)(l0 + l) * g.n + ((y0 - 1 + ly + N2) & (N2 - 1)) * N1 + ((x0 - 2 + 2 * q + N1) & (N1 - 1));
    sD[m] = (unsigned)__cvta_generic_to_shared(D + l * DPL + ly * DW + 2 * q);
    if (j < L * NCH && ((act >> l) & 1u)) vD |= 1u << m;
  }
  int poff = 0;
  unsigned psm = 0;
  if (t < NPC) {
    const int prow = t / (PW / 16), pq = t - prow * (PW / 16);
    poff = ((y0 - 1 + prow + N2) & (N2 - 1)) * N1 + ((x0 - 16 + 16 * pq + N1) & (N1 - 1));
    psm = (unsigned)__cvta_generic_to_shared(PH + prow * PW + 16 * pq);
  }
  constexpr unsigned SLOTD = L * DPL * 8;
  // node plane p of every active load + element layer p of the phase field into ring slot p
  auto issue_plane = [&](int p) {
    const unsigned slot = (p - zs + 1) & (RING - 1);
    const unsigned so = slot * SLOTD;
    if (DZ && (p <= 0 || p >= N3)) {  // fixed (zero) Dirichlet node planes z = 0, z = N3
#pragma unroll
      for (int m = 0; m < NDC; ++m)
        if ((vD >> m) & 1u)
          asm volatile("st.shared.v2.f64 [%0], {0d0000000000000000, 0d0000000000000000};\n" ::"r"(sD[m] + so)
                       : "memory");
    } else {
      const double* base = src + (long long)(DZ ? p - 1 : ((p + N3) & (N3 - 1))) * plane;
#pragma unroll
      for (int m = 0; m < NDC; ++m)
        if ((vD >> m) & 1u)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sD[m] + so), "l"(base + goffD[m]) : "memory");
    }
    if (t < NPC) {
      const uint8_t* pbase = cx.phase + (long long)((p + N3) & (N3 - 1)) * plane;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(psm + slot * PHS), "l"(pbase + poff) : "memory");
    }
  };
  double nb[NR + 2][3];
  auto readn = [&](int l, int p) {
    const double* Ds = D + ((p - zs + 1) & (RING - 1)) * (L * DPL) + l * DPL + NR * ty * DW + tx + 1;
#pragma unroll
    for (int a = 0; a < NR + 2; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) nb[a][b] = Ds[a * DW + b];
  };
  auto box = [&](double Qo[NR + 1][2]) {  // x pairs, then (x, y) quads of the plane just read
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
  auto kap = [&](int layer, double a[NR + 1][2]) {  // kappa (x h/12) of the 3 x 2 elements of `layer`
    const unsigned char* Pl = PH + ((layer - zs + 1) & (RING - 1)) * PHS + NR * ty * PW + tx + 15;
#pragma unroll
    for (int e = 0; e < NR + 1; ++e) {
      a[e][0] = Pl[e * PW] ? k1 : k0;
      a[e][1] = Pl[e * PW + 1] ? k1 : k0;
    }
  };
  // per-node kappa sums of one layer: all 4 elements, the 2 with x offset 0, the 2 with y offset 0
  auto ksums = [&](const double a[NR + 1][2], double K4[NR], double Kx[NR], double Ky[NR]) {
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      K4[m] = (a[m][0] + a[m][1]) + (a[m + 1][0] + a[m + 1][1]);
      Kx[m] = a[m][1] + a[m + 1][1];
      Ky[m] = a[m + 1][0] + a[m + 1][1];
    }
  };
  // start p of plane j: 5 d sum_e kappa + in-plane edge terms + its z- neighbour (plane j-1),
  //   Kx+ xp + (Ks - Kx+) xm + Ky+ yp + (Ks - Ky+) ym + 5 Ks d + Klo d_{j-1}
  //   = Kx+ (xp - xm) + Ky+ (yp - ym) + Ks (xm + ym + 5 d) + Klo d_{j-1}
  // with Ks, Kx+, Ky+ the node sums over both layers (load independent, computed once a step).
  auto start_p = [&](const double Ks[NR], const double Kxp[NR], const double Kyp[NR], const double Klo[NR],
                     const double cprev[NR], double pp[NR]) {
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      const double t3 = fma(5.0, nb[m + 1][1], nb[m + 1][0] + nb[m][1]);
      double E = Kxp[m] * (nb[m + 1][2] - nb[m + 1][0]);
      E = fma(Kyp[m], nb[m + 2][1] - nb[m][1], E);
      E = fma(Ks[m], t3, E);
      pp[m] = fma(Klo[m], cprev[m], E);
    }
  };
  auto nodesums = [&](const double Klo[NR], const double Kxlo[NR], const double Kylo[NR], const double Khi[NR],
                      const double Kxhi[NR], const double Kyhi[NR], double Ks[NR], double Kxp[NR], double Kyp[NR]) {
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      Ks[m] = Klo[m] + Khi[m];
      Kxp[m] = Kxlo[m] + Kxhi[m];
      Kyp[m] = Kylo[m] + Kyhi[m];
    }
  };
#pragma unroll 1
  for (int p = zs - 1; p <= zs + LA - 1; ++p) {
    if (p <= ze) issue_plane(p);
    cp_commit();
  }
  cp_wait<LA - 1>();
  __syncthreads();
  KMLState<L> A, B;
  {  // planes zs-1 and zs: quads, the layer zs-1 box sums and the partial p of plane zs
    double al[NR + 1][2], ah[NR + 1][2], Khi[NR], Kxhi[NR], Kyhi[NR], Ks[NR], Kxp[NR], Kyp[NR];
    kap(zs - 1, al);
    kap(zs, ah);
    ksums(al, A.Klo, A.Kxlo, A.Kylo);
    ksums(ah, Khi, Kxhi, Kyhi);
    nodesums(A.Klo, A.Kxlo, A.Kylo, Khi, Kxhi, Kyhi, Ks, Kxp, Kyp);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      // every load slot is computed (no per-load branch: the loads interleave for ILP); a frozen
      // or absent load only has its stores and partial suppressed
      double Qm[NR + 1][2], cprev[NR];
      readn(l, zs - 1);
      box(Qm);
#pragma unroll
      for (int m = 0; m < NR; ++m) cprev[m] = nb[m + 1][1];
      readn(l, zs);
      box(A.Qk[l]);
      double KS[NR + 1];
#pragma unroll
      for (int e = 0; e < NR + 1; ++e)
        KS[e] = fma(al[e][0], Qm[e][0] + A.Qk[l][e][0], al[e][1] * (Qm[e][1] + A.Qk[l][e][1]));
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        A.KSlo[l][m] = KS[m] + KS[m + 1];
        A.cp[l][m] = nb[m + 1][1];
      }
      start_p(Ks, Kxp, Kyp, A.Klo, cprev, A.pp[l]);
    }
#pragma unroll
    for (int m = 0; m < NR; ++m) {  // the step reading plane zs + 1 carries layer zs
      A.Klo[m] = Khi[m];
      A.Kxlo[m] = Kxhi[m];
      A.Kylo[m] = Kyhi[m];
    }
  }
  double part[L];
#pragma unroll
  for (int l = 0; l < L; ++l) part[l] = 0.0;
  double* outp = dst + (long long)(y0 + NR * ty) * N1 + (x0 + tx);
  // the step reading node plane j (zs < j <= ze): completes p of plane j-1, starts p of plane j
  auto step = [&](int j, const KMLState<L>& I, KMLState<L>& O) {
    if (j - 1 + LA <= ze) issue_plane(j - 1 + LA);
    cp_commit();
    cp_wait<LA - 1>();
    __syncthreads();
    double al[NR + 1][2], ah[NR + 1][2];
    kap(j - 1, al);  // layer j-1: per-element kappa of the box term (its node sums are I.K*lo)
    kap(j, ah);
    double Khi[NR], Kxhi[NR], Kyhi[NR], Ks[NR], Kxp[NR], Kyp[NR];
    ksums(ah, Khi, Kxhi, Kyhi);
    nodesums(I.Klo, I.Kxlo, I.Kylo, Khi, Kxhi, Kyhi, Ks, Kxp, Kyp);
    const long long orow = (long long)(j - 1 - dz) * plane;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      readn(l, j);
      box(O.Qk[l]);
      double KS[NR + 1];
#pragma unroll
      for (int e = 0; e < NR + 1; ++e)
        KS[e] = fma(al[e][0], I.Qk[l][e][0] + O.Qk[l][e][0], al[e][1] * (I.Qk[l][e][1] + O.Qk[l][e][1]));
      double* op = outp + (long long)(l0 + l) * g.n + orow;
#pragma unroll
      for (int m = 0; m < NR; ++m) {
        const double KShi = KS[m] + KS[m + 1];
        const double pv = fma(I.Klo[m], nb[m + 1][1], I.pp[l][m]) - (I.KSlo[l][m] + KShi);
        if ((act >> l) & 1u) op[m * N1] = pv;
        part[l] = fma(I.cp[l][m], pv, part[l]);
        O.KSlo[l][m] = KShi;
        O.cp[l][m] = nb[m + 1][1];
      }
      start_p(Ks, Kxp, Kyp, I.Klo, I.cp[l], O.pp[l]);
    }
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      O.Klo[m] = Khi[m];
      O.Kxlo[m] = Kxhi[m];
      O.Kylo[m] = Kyhi[m];
    }
  };
  int j = zs + 1;
#pragma unroll 1
  for (; j + 1 <= ze; j += 2) {  // unrolled by two: the carried state ping-pongs A <-> B
    step(j, A, B);
    step(j + 1, B, A);
  }
  if (j <= ze) step(j, A, B);
  cp_wait<0>();
  const int my = (zcI * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
  for (int l = 0; l < L; ++l)
    if ((act >> l) & 1u) dp_finish(cx, l0 + l, 0, my, part[l], red_sh, mode);
}

// Multi-load thermal K for 3D grids with N1 >= 32, N2 >= 16 (periodic or Dirichlet z); -1 if the
// grid needs another kernel (slab halos, all-Dirichlet storage, small grids).  CTA partials of d.p
// are indexed like the one-load 32 x 16 tile kernel (same nblk for the scalar kernel).
int launch_kp_thermal_ml(const Ctx& cx, int mode, const double* src, double* dst, cudaStream_t s) {
  const Geo& g = cx.g;
  if (g.dim != 3 || g.c != 1 || g.N1 < 32 || g.N2 < 16 || g.halo || g.dir3 || g.dmask) return -1;
  const int ZC = g.KZC;
  const int nzc = (g.P3 + ZC - 1) / ZC;
  const int L = g.nrhs >= KML_LMAX ? KML_LMAX : g.nrhs;
  const int ngrp = (g.nrhs + L - 1) / L;
  const dim3 grid(g.N1 / KML_TX, g.N2 / KML_TH, nzc * ngrp);
  const int sm = kml_smem_bytes(L);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    kern<<<grid, KML_T, sm, s>>>(cx, mode, src, dst, ZC);
  };
  if (g.dirz) {
    if (L == 1) go(kp_thermal3d_ml_kernel<1, true>);
    else if (L == 2) go(kp_thermal3d_ml_kernel<2, true>);
    else go(kp_thermal3d_ml_kernel<3, true>);
  } else {
    if (L == 1) go(kp_thermal3d_ml_kernel<1, false>);
    else if (L == 2) go(kp_thermal3d_ml_kernel<2, false>);
    else go(kp_thermal3d_ml_kernel<3, false>);
  }
  return 1;
}

}  // namespace uno
