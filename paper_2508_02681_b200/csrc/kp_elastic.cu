// kp_elastic.cu — matrix-free Q1 elasticity K.u (Eq 22 with D of Eq 80) in the
// Walsh-Hadamard modal basis of the element (elastic_modal.cuh).
//
// Per element: forward 8-point WHT of the corner displacements (3 components), the 45-entry
// sparse modal operator (lam, mu of the element's phase), inverse WHT: ~240 flops instead of the
// 576 FMAs of the dense 24x24 element matrix.  Node-centric gather without atomics: a CTA owns a
// 16 x 8 node tile marching over z; each z step computes the 17 x 9 element layer above the
// current node plane once (160 threads, one element column each).  A thread keeps its element
// column's upper corner values and upper-face outputs in registers for the next layer, so a layer
// reads one node plane of the tile from shared memory and stores only the plane's combined outputs
// (lower faces of this layer + upper faces of the previous one); every node then sums its 4 (x, y)
// element columns.  d planes stream through a 4-slot cp.async ring (planes k+2, k+3 in flight while
// layer k is computed).
#include <cuda_runtime.h>

#include "common.cuh"
#include "dev_common.cuh"
#include "elastic_modal.cuh"
#include "kernels.cuh"

namespace uno {

constexpr int KM_TX = 16, KM_TY = 8, KM_T = 160;
// node tile x0-2 .. x0+17 (20 wide: 16-byte aligned pairs; x0-2 is unused) by y0-1 .. y0+8
constexpr int KM_DW = KM_TX + 4, KM_DH = KM_TY + 2, KM_DP = KM_DW * KM_DH;
constexpr int KM_EW = KM_TX + 1, KM_EH = KM_TY + 1, KM_NE = KM_EW * KM_EH;  // 17 x 9 elements
constexpr int KM_RING = 8, KM_LA = 4;  // ring slots; planes prefetched ahead
constexpr int KM_PLANE = 3 * KM_DP;                 // doubles per ring slot (3 components)
constexpr int KM_NCH = KM_PLANE / 2;                 // 16-byte chunks per ring slot
constexpr int KM_NCP = (KM_NCH + KM_T - 1) / KM_T;    // cp.async per thread per plane

__host__ __device__ constexpr int km_smem_bytes() {
  return (KM_RING * KM_PLANE + 2 * 12 * KM_NE) * (int)sizeof(double);
}

__global__ void __launch_bounds__(KM_T, 3) kp_elastic3d_modal_kernel(Ctx cx, int mode, const double* __restrict__ src,
                                                                     double* __restrict__ dst, int ZC) {
  const Geo g = cx.g;
  const int nzc = (g.P3 + ZC - 1) / ZC;
  const int load = blockIdx.z / nzc;
  const int zcI = blockIdx.z - load * nzc;
  if (mode == CG && !cx.st[load].active) return;
  const int dz = g.dirz;
  extern __shared__ double kms[];
  double* D = kms;                           // [RING][3][10][20]
  double* Lb0 = D + KM_RING * KM_PLANE;      // [2][12][NE] node-plane outputs, double-buffered by layer parity
  __shared__ double red_sh[32];
  const int t = threadIdx.x;
  const int N1 = g.N1, N2 = g.N2, N3 = g.N3;
  const long long n = g.n;
  const long long plane = (long long)N1 * N2;
  const int x0 = blockIdx.x * KM_TX, y0 = blockIdx.y * KM_TY;
  const int zs = zcI * ZC + dz + g.zlo, ze = min(zs + ZC, g.P3 + dz + g.zlo);  // slab: global planes
  const double* dv = cg_dir(cx, mode, src, load) + (long long)load * 3 * n;
  const double hs = g.h / (72.0 * 64.0);
  const double l0 = cx.mat[0][0] * hs, m0 = cx.mat[0][1] * hs, l1 = cx.mat[1][0] * hs, m1 = cx.mat[1][1] * hs;
  // copy assignment of the 3 x 10 x 20 plane tile in 16-byte pairs (clamped: harmless duplicates)
  long long goff[KM_NCP];  // in-plane offset
  int gcomp[KM_NCP];
  unsigned sdst[KM_NCP];
#pragma unroll
  for (int m = 0; m < KM_NCP; ++m) {
    const int j = min(t + m * KM_T, KM_NCH - 1);
    const int comp = j / (KM_DP / 2), r = j - comp * (KM_DP / 2);
    const int ly = r / (KM_DW / 2), lx = 2 * (r - ly * (KM_DW / 2));
    gcomp[m] = comp;
    goff[m] = (long long)((y0 - 1 + ly + N2) & (N2 - 1)) * N1 + ((x0 - 2 + lx + N1) & (N1 - 1));
    sdst[m] = (unsigned)__cvta_generic_to_shared(D + comp * KM_DP + ly * KM_DW + lx);
  }
  auto slot_of = [&](int p) { return (p - zs + 1) & (KM_RING - 1); };
  auto issue_plane = [&](int p) {
    const unsigned so = slot_of(p) * KM_PLANE * 8;
    if (dz && (p <= 0 || p >= N3)) {
#pragma unroll
      for (int m = 0; m < KM_NCP; ++m)
        asm volatile("st.shared.v2.f64 [%0], {0d0000000000000000, 0d0000000000000000};\n" ::"r"(sdst[m] + so)
                     : "memory");
    } else {
      // component c of plane p starts at base + c * cst (slab halo buffers: [nrhs][3][N2][N1])
      const double* base;
      long long cst = n;
      if (g.halo && (p < g.zlo || p >= g.zlo + g.P3)) {
        base = (p < g.zlo ? cx.hlo : cx.hhi) + (long long)load * 3 * plane;
        cst = plane;
      } else {
        base = dv + (long long)(g.halo ? p - g.zlo : (dz ? p - 1 : ((p + N3) & (N3 - 1)))) * plane;
      }
#pragma unroll
      for (int m = 0; m < KM_NCP; ++m)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst[m] + so),
                     "l"(base + gcomp[m] * cst + goff[m])
                     : "memory");
    }
  };
  // element column owned by this thread: the plane-(k+1) corner values (uc) and the upper-face
  // outputs (vc) of layer k stay in registers for layer k+1, so a layer reads one node plane from
  // smem and writes only the combined lower-face outputs Lb = v_lower(k) + v_upper(k-1).
  const bool eth = t < KM_NE;
  const int exl = eth ? t % KM_EW : 0, eyl = eth ? t / KM_EW : 0;
  const long long pbase = (long long)((y0 - 1 + eyl + N2) & (N2 - 1)) * N1 + ((x0 - 1 + exl + N1) & (N1 - 1));
  // uc = 2D (x, y) Walsh-Hadamard modes of the plane-(k+1) corners, vc = the upper-face output
  // modes of layer k: the 8-point WHT of a layer is the z butterfly of its two planes' 2D modes
  // (the x and y butterflies of a shared node plane are done once), and the output plane k is one
  // 2D inverse of (lower-face modes of layer k + upper-face modes of layer k-1).
  double uc[12], vc[12];
  auto read_corners = [&](int p, double* dstv) {  // the 4 (x, y) corners of node plane p
    const double* Dp = D + slot_of(p) * KM_PLANE + eyl * KM_DW + exl + 1;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int al = 0; al < 3; ++al) dstv[3 * a + al] = Dp[al * KM_DP + ((a >> 1) & 1) * KM_DW + (a & 1)];
  };
  // phase byte of element layer k, loaded three layers ahead (a queue of 3 registers): one layer
  // ahead left 13 % of the stall samples on the load (ncu round 2)
  auto phase_raw = [&](int k) -> unsigned {
    // Dirichlet z: the prefetches past the last layer (N3 ...) do not exist — clamp the address
    // (their values are never used); a predicated load would cost the prefetch its early issue
    const int layer = dz ? min(k, N3 - 1) : ((k + N3) & (N3 - 1));
    return __ldg(cx.phase + (long long)layer * plane + pbase);
  };
  unsigned ph0 = phase_raw(zs - 1), ph1 = phase_raw(zs), ph2 = phase_raw(zs + 1);
  auto element_layer = [&](int k, bool want_lower) {  // element layer between node planes k, k+1
    const bool ph = ph0 != 0;
    ph0 = ph1;
    ph1 = ph2;
    ph2 = phase_raw(k + 3);
    if (!eth) return;
    const double ls = ph ? l1 : l0, ms = ph ? m1 : m0;
    double w[12];
    read_corners(k + 1, w);
#pragma unroll
    for (int al = 0; al < 3; ++al) modal::wht4(w + al);
    double u[24];  // modes m (z bit clear) = lower + upper, m | 4 = lower - upper
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      u[i] = uc[i] + w[i];
      u[12 + i] = uc[i] - w[i];
      uc[i] = w[i];
    }
    double v[24];
    modal::apply_blocked(v, u, ls, ms);  // rows of mode 0 are zero
    double o[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      o[i] = (v[i] + v[12 + i]) + vc[i];
      vc[i] = v[i] - v[12 + i];
    }
    if (want_lower) {
#pragma unroll
      for (int al = 0; al < 3; ++al) modal::wht4(o + al);
#pragma unroll
      for (int i = 0; i < 12; ++i) Lb0[((k & 1) * 12 + i) * KM_NE + t] = o[i];
    }
  };
  // prologue: planes zs-1 .. zs+3 in flight; element layer zs-1 (its upper faces feed plane zs)
#pragma unroll 1
  for (int p = zs - 1; p <= zs - 1 + KM_LA; ++p) {
    if (p <= ze) issue_plane(p);
    cp_commit();
  }
  cp_wait<KM_LA - 1>();  // planes zs-1, zs
  __syncthreads();
  if (eth) {
    read_corners(zs - 1, uc);
#pragma unroll
    for (int al = 0; al < 3; ++al) modal::wht4(uc + al);
  }
#pragma unroll
  for (int i = 0; i < 12; ++i) vc[i] = 0.0;
  element_layer(zs - 1, false);
  cp_wait<KM_LA - 2>();  // plane zs+1 (read by the first layer of the loop)
  __syncthreads();
  const bool nth = t < KM_TX * KM_TY;
  const int tx = t % KM_TX, ty = t / KM_TX;
  double part = 0.0;
  // One barrier per layer: it publishes this layer's outputs (Lb, double-buffered by parity so the
  // next layer may be written while slow threads still gather this one), makes plane k+2 visible
  // for the next layer, and frees the slot refilled with plane k+4 (last read four layers ago).
#pragma unroll 1
  for (int k = zs; k < ze; ++k) {
    element_layer(k, true);
    cp_wait<KM_LA - 3>();  // plane k+2 landed (k+3 may still be in flight)
    __syncthreads();
    if (k + KM_LA <= ze) issue_plane(k + KM_LA);
    cp_commit();
    if (nth) {
      const double* Lb = Lb0 + (k & 1) * 12 * KM_NE;
      double p[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int ox = o & 1, oy = o >> 1;
        const int e = (ty + oy) * KM_EW + tx + ox;
        const int a = (1 - ox) + 2 * (1 - oy);  // the node's corner in the element
#pragma unroll
        for (int al = 0; al < 3; ++al) p[al] += Lb[(3 * a + al) * KM_NE + e];
      }
      const double* Dc = D + slot_of(k) * KM_PLANE + (ty + 1) * KM_DW + tx + 2;
      const long long gi = (long long)(k - dz - g.zlo) * plane + (long long)(y0 + ty) * N1 + x0 + tx;
      if ((g.dir3 && (x0 + tx == 0 || y0 + ty == 0 || k == 0)) || (g.zpad && k == 0))
        p[0] = p[1] = p[2] = 0.0;  // Dirichlet nodes (all-Dirichlet storage / slab Dirichlet-z face)
#pragma unroll
      for (int al = 0; al < 3; ++al) {
        dst[(long long)load * 3 * n + al * n + gi] = p[al];
        part = fma(Dc[al * KM_DP], p[al], part);
      }
    }
  }
  cp_wait<0>();
  const int nblk = gridDim.x * gridDim.y * nzc;
  const int my = (zcI * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  dp_finish(cx, load, nblk, my, part, red_sh, mode);
}

int launch_kp_elastic_modal(const Ctx& cx, int mode, const double* src, double* dst, cudaStream_t s) {
  const Geo& g = cx.g;
  if (g.dim != 3 || g.c != 3 || g.N1 < KM_TX || g.N2 < KM_TY) return -1;
  const int ZC = g.KZC;
  const dim3 grid(g.N1 / KM_TX, g.N2 / KM_TY, ((g.P3 + ZC - 1) / ZC) * g.nrhs);
  const int sm = km_smem_bytes();
  // the attribute is per device: set it on every launch (cheap), like set_smem in kernels.cu
  cudaFuncSetAttribute(kp_elastic3d_modal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  kp_elastic3d_modal_kernel<<<grid, KM_T, sm, s>>>(cx, mode, src, dst, ZC);
  return 1;
}

int kp_elastic_modal_nblk(const Geo& g) {
  const int ZC = g.KZC;
  return (g.N1 / KM_TX) * (g.N2 / KM_TY) * ((g.P3 + ZC - 1) / ZC);
}

}  // namespace uno
