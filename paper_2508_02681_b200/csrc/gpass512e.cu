// gpass512e.cu — elastic G pass at N3 = 512 (config 4: 512^3, c = 3, periodic z), persistent CTAs.
// z FFT -> s_hat = G_hat r_hat (3x3 real-symmetric block per bin, Eq 46/49, App. B) and the
// Parseval partial of gamma_1 -> inverse z FFT (Alg 2 l.4-7), in place on the half
// spectrum [load][c][kx][z][y].
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"
#include "dev_common.cuh"

namespace uno {

// Elastic G pass at N3 = 512 (config 4), persistent: the three 64 KB component tiles (8 y columns
// x 512 z each) fill the SM's shared memory (one CTA per SM), so load / compute / store can only
// overlap inside the CTA.  Each CTA walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...; as soon as
// component q of the current tile has been stored, the cp.async copies of component q of the NEXT
// tile start into the same buffer (one commit group per component) and a third of the next tile's
// symbol rows is prefetched into L2 — they land while the inverse stages of the other components,
// the stores and the next tile's first forward stages run.
// 256 threads, two radix-8 butterflies per thread in every Stockham stage (512 = 8 . 8 . 8): the
// fused middle stage (last forward stage -> 3x3 symbol multiply -> first inverse stage, all on
// registers) holds 3 components x 8 bins x 2 items = 192 registers of data, which fits the
// 255-register budget of a 256-thread CTA without spills; with 512 threads and 128 registers the
// same stage spills, and the local-memory traffic (only ~28 KB of L1 is left next to 200 KB of
// shared memory) cost more than the pipelining gained (measured: 3.70 ms vs 3.45 ms one tile per
// CTA).  Same tile shape and per-tile gamma partials as gpass_z_kernel<512, 3>.
#ifndef UNO_G512E_PERSIST
#define UNO_G512E_PERSIST 1  // 0: A/B builds only (the one-tile-per-CTA gpass_z_kernel<512, 3>)
#endif
#ifndef UNO_G5E_W
#define UNO_G5E_W 8
#endif
#ifndef UNO_G5E_SYM
#define UNO_G5E_SYM 0  // symbol loads: 0 at the item start, 1 half an item ahead (first before the last forward stage), 2 first at item 0
#endif
constexpr int kG512ePersistCTAs = 148;
namespace g5e {
constexpr int W = UNO_G5E_W;  // y columns per tile (8: one CTA per SM; 4: two)
constexpr int L = 512, NC = 3, T = 32 * W, R = 8, NJ = L / R, NH = NJ * W / T;  // NH = 2 items per thread
constexpr int TJ = T / W;        // items j0 .. j0 + TJ - 1 per round
__device__ __forceinline__ int tix(int j, int c) { return W == 8 ? tidx(j, c) : tidx_w<W>(j, c); }
static_assert(NH == 2 && pick_radix(512) == 8 && pick_radix(64) == 8 && pick_radix(8) == 8, "512 = 8.8.8");

struct Args {
  double2* spec;       // component 0 of this load
  const double* gtab;  // symbol entries [6][nspec]
  long long nspec;
  int N2, N3, M, ntile_y;
};
__device__ __forceinline__ long long tile_off(const Args& a, int tile) {
  const int kx = tile / a.ntile_y;
  return (long long)kx * a.N3 * a.N2 + (tile - kx * a.ntile_y) * W;
}
// copies of component q of the tile at boff (one commit group) + symbol entries 2q, 2q + 1 -> L2
template <int T>
__device__ __forceinline__ void issue_t(const Args& a, double2* tile_q, int q, long long boff) {
  constexpr int L = 512;
  const int t = threadIdx.x;
  const double2* base = a.spec + q * a.nspec + boff;
#pragma unroll
  for (int i = 0; i < W * L / T; ++i) {
    const int e = t + i * T;
    cp_async16(&tile_q[tix(e / W, e % W)], base + (long long)(e / W) * a.N2 + (e % W));
  }
  cp_commit();
#pragma unroll
  for (int i = 0; i < 2 * L / T; ++i) {
    const int r = t + i * T, ent = 2 * q + r / L, kz = r & (L - 1);
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a.gtab + ent * a.nspec + boff + (long long)kz * a.N2));
  }
}
// One radix-8 Stockham stage of span NS over the 8 columns of one component tile, in place
// (fft.cuh fft_stage with two items per thread: j = t / 8 and t / 8 + 32).
template <int NS, bool INV>
__device__ __forceinline__ void stage(double2* s, const double2* __restrict__ tw) {
  const int t = threadIdx.x, c = t % W, j0 = t / W;
  double2 v[NH][R];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * TJ, k = j % NS;
#pragma unroll
    for (int r = 0; r < R; ++r) v[h][r] = s[tix(j + r * NJ, c)];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = tw[r * k * (L / (NS * R))];
        if (INV) w.y = -w.y;
        v[h][r] = cmul(v[h][r], w);
      }
    }
    dft_reg<R, INV>(v[h]);
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * TJ, k = j % NS, base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) s[tix(base + r * NS, c)] = v[h][r];
  }
  __syncthreads();
}

// First inverse stage after the middle (span R): item j reads canonical rows p = j + r NJ, which
// the middle stage left at row (p >> 3) + NJ (p & 7) (see tile_pass), and writes canonical rows.
__device__ __forceinline__ void stage_inv_rot(double2* s, const double2* __restrict__ tw) {
  constexpr int NS = R;
  const int t = threadIdx.x, c = t % W, j0 = t / W;
  double2 v[NH][R];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * TJ, k = j % NS, row0 = (j >> 3) + NJ * (j & 7);
#pragma unroll
    for (int r = 0; r < R; ++r) v[h][r] = s[tix(row0 + 8 * r, c)];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      double2 w = tw[r * k * (L / (NS * R))];
      w.y = -w.y;
      v[h][r] = cmul(v[h][r], w);
    }
    dft_reg<R, true>(v[h]);
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * TJ, k = j % NS, base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) s[tix(base + r * NS, c)] = v[h][r];
  }
  __syncthreads();
}

// symbol entries (Eq B7 order, dev_common.cuh gmul_vals) of the bins j + r NJ, r = R0 .. R0 + 3
template <int R0>
__device__ __forceinline__ void load_sym(double (&sy)[4][6], const double* __restrict__ gtab, long long nspec,
                                         long long bcol, int j, int N2) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double* p = gtab + bcol + (long long)(j + (R0 + r) * NJ) * N2;
#pragma unroll
    for (int e = 0; e < 6; ++e) sy[r][e] = __ldg(p + e * nspec);
  }
}
// s_hat = G_hat r_hat on one bin and its Parseval term (same operation order as gmul_vals<3>)
__device__ __forceinline__ double gmul3(double2& x1, double2& x2, double2& x3, const double (&g)[6], double w) {
  const double v1 = g[0], v2 = g[1], v3 = g[2], v4 = g[3], v5 = g[4], v6 = g[5];
  const double2 X1 = x1, X2 = x2, X3 = x3;
  double2 Y1, Y2, Y3;
  Y1.x = fma(v1, X1.x, fma(v3, X2.x, v6 * X3.x));
  Y1.y = fma(v1, X1.y, fma(v3, X2.y, v6 * X3.y));
  Y2.x = fma(v3, X1.x, fma(v2, X2.x, v5 * X3.x));
  Y2.y = fma(v3, X1.y, fma(v2, X2.y, v5 * X3.y));
  Y3.x = fma(v6, X1.x, fma(v5, X2.x, v4 * X3.x));
  Y3.y = fma(v6, X1.y, fma(v5, X2.y, v4 * X3.y));
  x1 = Y1;
  x2 = Y2;
  x3 = Y3;
  return w * (X1.x * Y1.x + X1.y * Y1.y + X2.x * Y2.x + X2.y * Y2.y + X3.x * Y3.x + X3.y * Y3.y);
}

// One tile.  Forward stages (span 1, R) per component as its copy group lands; middle stage per
// item (j, c) entirely on the item's own rows: the last forward stage (span NJ) reads and writes
// rows j + r NJ, the symbol multiply acts on those bins, and the first inverse stage (span 1)
// reads the same rows — its outputs (canonical rows R j + r) are parked in the rows the item owns
// (row j + r NJ holds canonical row R j + r), so no other item's data is touched, one item is in
// registers at a time (96 data registers) and the next inverse stage reads through that
// permutation (stage_inv_rot).  The registers this frees hold the item's 48 symbol entries, loaded
// half an item ahead (the loads of item 0 are issued before the last forward stage of component
// 2), so the multiply does not wait on L2.  Not inlined: nothing of a tile's index arithmetic is
// hoisted out of the persistent loop.
__device__ __noinline__ double tile_pass(Args a, int tile, int next) {
  extern __shared__ double2 smem[];
  double2* tiles[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) tiles[q] = smem + q * W * L;
  const double2* tw = smem + NC * W * L;
  const int t = threadIdx.x, c = t % W, j0 = t / W;
  const long long boff = tile_off(a, tile);
  const double w = parseval_w(tile / a.ntile_y, a.M);
  double sa[4][6], sb[4][6];  // symbol entries of bins r = 0..3 / 4..7 of the current item
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    // component q's copy group has landed (groups are committed in component order)
    if (q == 0) cp_wait<2>();
    else if (q == 1) cp_wait<1>();
    else cp_wait<0>();
    __syncthreads();
    stage<1, false>(tiles[q], tw);
#if UNO_G5E_SYM == 1
    if (q == NC - 1) {
      load_sym<0>(sa, a.gtab, a.nspec, boff + c, j0, a.N2);
      load_sym<4>(sb, a.gtab, a.nspec, boff + c, j0, a.N2);
    }
#endif
    stage<R, false>(tiles[q], tw);
  }
  double part = 0.0;
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * TJ;
    double2 v[NC][R];
#if UNO_G5E_SYM == 0
    load_sym<0>(sa, a.gtab, a.nspec, boff + c, j, a.N2);
    load_sym<4>(sb, a.gtab, a.nspec, boff + c, j, a.N2);
#elif UNO_G5E_SYM == 2
    if (h == 0) {
      load_sym<0>(sa, a.gtab, a.nspec, boff + c, j, a.N2);
      load_sym<4>(sb, a.gtab, a.nspec, boff + c, j, a.N2);
    }
#endif
#pragma unroll
    for (int q = 0; q < NC; ++q) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = tiles[q][tix(j + r * NJ, c)];
#pragma unroll
      for (int r = 1; r < R; ++r) v[q][r] = cmul(v[q][r], tw[r * j]);
      Dft<R>::run(v[q]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) part += gmul3(v[0][r], v[1][r], v[2][r], sa[r], w);
#if UNO_G5E_SYM >= 1
    if (h + 1 < NH) load_sym<0>(sa, a.gtab, a.nspec, boff + c, j + T / 8, a.N2);
#endif
#pragma unroll
    for (int r = 0; r < 4; ++r) part += gmul3(v[0][4 + r], v[1][4 + r], v[2][4 + r], sb[r], w);
#if UNO_G5E_SYM >= 1
    if (h + 1 < NH) load_sym<4>(sb, a.gtab, a.nspec, boff + c, j + T / 8, a.N2);
#endif
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      dft_reg_inv_inline<R>(v[q]);
#pragma unroll
      for (int r = 0; r < R; ++r) tiles[q][tix(j + r * NJ, c)] = v[q][r];  // canonical row R j + r, parked
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    stage_inv_rot(tiles[q], tw);
    // last inverse stage (span NJ): item j reads and produces rows j + r NJ, so its outputs go
    // straight to the spectrum (8 columns = 128 contiguous bytes per row) without another
    // shared-memory round trip
    {
      double2* base = a.spec + q * a.nspec + boff + c;
      double2 v[NH][R];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int j = j0 + h * TJ;
#pragma unroll
        for (int r = 0; r < R; ++r) v[h][r] = tiles[q][tix(j + r * NJ, c)];
#pragma unroll
        for (int r = 1; r < R; ++r) v[h][r] = cmul(v[h][r], cconj(tw[r * j]));
        dft_reg<R, true>(v[h]);
      }
      __syncthreads();  // every thread has read its part of tiles[q]: the buffer is free
      if (next >= 0) issue_t<T>(a, tiles[q], q, tile_off(a, next));
      else cp_commit();
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int j = j0 + h * TJ;
#pragma unroll
        for (int r = 0; r < R; ++r) base[(long long)(j + r * NJ) * a.N2] = v[h][r];
      }
    }
  }
  return part;
}
}  // namespace g5e

// ---- TMA variant of the 256-thread kernel: the component tiles move by cp.async.bulk.tensor
// (one elected thread, two 256-row boxes per component; CU_TENSOR_MAP_SWIZZLE_128B is exactly
// fft.cuh's tidx swizzle: 16-byte chunk c of row j at chunk c ^ (j & 7)), so the compute threads
// issue no global loads or stores for the tiles: in the cp.async version the 16 ST.E.128 + 16
// LDGSTS per thread at the end of every component sat in the same in-order LSU queue as the next
// stage's LDS (ncu: 13 % of the stall samples on those, mio_throttle 18 %).  Loads complete on
// one mbarrier per component buffer; a buffer is reloaded one phase after its store was issued
// (cp.async.bulk.wait_group.read), the symbol rows of the next tile are prefetched into L2 with
// cp.async.bulk.prefetch.tensor.
namespace g5t {
using g5e::Args;
using g5e::gmul3;
using g5e::load_sym;
using g5e::stage;
using g5e::stage_inv_rot;
constexpr int L = 512, NC = 3, T = 256, R = 8, NJ = L / R, NH = g5e::NH;
constexpr unsigned kCompBytes = 8 * L * 16;

__device__ __forceinline__ unsigned sm_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned mb, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "G5T_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra G5T_DONE;\n"
      "bra G5T_WAIT;\n"
      "G5T_DONE:\n"
      "}\n" ::"r"(mb),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load(unsigned dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3, unsigned mb) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mb)
      : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* tm, int c0, int c1, int c2, int c3, unsigned src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(tm), "r"(c0),
               "r"(c1), "r"(c2), "r"(c3), "r"(src)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* tm, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];\n" ::"l"(tm), "r"(c0), "r"(c1), "r"(c2),
               "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}

struct Tma {
  const CUtensorMap* spec;  // doubles [load * c + q][kx][z][2 y], box 16 x 256, SWIZZLE_128B
  const CUtensorMap* sym;   // doubles [entry][kx][z][y], box 8 x 256 (L2 prefetch only)
  unsigned tiles, mbar;     // shared-memory addresses of tile 0 and of the three mbarriers
  int lc0;                  // load * c
};
// component q of `tile` -> its buffer (thread 0); also the L2 prefetch of symbol entries 2q, 2q + 1
__device__ __forceinline__ void load_comp(const Tma& m, const Args& a, int q, int tile) {
  const int kx = tile / a.ntile_y, y0 = (tile - kx * a.ntile_y) * 8;
  const unsigned mb = m.mbar + 8 * q, dst = m.tiles + q * kCompBytes;
  mbar_expect_tx(mb, kCompBytes);
  tma_load(dst, m.spec, 2 * y0, 0, kx, m.lc0 + q, mb);
  tma_load(dst + kCompBytes / 2, m.spec, 2 * y0, L / 2, kx, m.lc0 + q, mb);
#pragma unroll
  for (int e = 2 * q; e < 2 * q + 2; ++e) {
    tma_prefetch(m.sym, y0, 0, kx, e);
    tma_prefetch(m.sym, y0, L / 2, kx, e);
  }
}

__device__ __noinline__ double tile_pass(Args a, Tma m, int tile, int next, int it) {
  extern __shared__ __align__(1024) double2 smem[];
  double2* tiles[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) tiles[q] = smem + q * 8 * L;
  const double2* tw = smem + NC * 8 * L;
  const int t = threadIdx.x, c = t & 7, j0 = t >> 3;
  const int kx = tile / a.ntile_y, y0 = (tile - kx * a.ntile_y) * 8;
  const long long boff = (long long)kx * a.N3 * a.N2 + y0;
  const double w = parseval_w(kx, a.M);
  double sa[4][6], sb[4][6];
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    mbar_wait(m.mbar + 8 * q, it & 1);
    stage<1, false>(tiles[q], tw);
    stage<R, false>(tiles[q], tw);
    if (q == 0 && it > 0 && t == 0) {  // buffer 2 of this tile: its store (previous tile) was the last one issued
      bulk_wait_read<0>();
      load_comp(m, a, 2, tile);
    }
  }
  double part = 0.0;
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = j0 + h * (T / 8);
    double2 v[NC][R];
    load_sym<0>(sa, a.gtab, a.nspec, boff + c, j, a.N2);
    load_sym<4>(sb, a.gtab, a.nspec, boff + c, j, a.N2);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = tiles[q][tidx(j + r * NJ, c)];
#pragma unroll
      for (int r = 1; r < R; ++r) v[q][r] = cmul(v[q][r], tw[r * j]);
      Dft<R>::run(v[q]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) part += gmul3(v[0][r], v[1][r], v[2][r], sa[r], w);
#pragma unroll
    for (int r = 0; r < 4; ++r) part += gmul3(v[0][4 + r], v[1][4 + r], v[2][4 + r], sb[r], w);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      dft_reg_inv_inline<R>(v[q]);
#pragma unroll
      for (int r = 0; r < R; ++r) tiles[q][tidx(j + r * NJ, c)] = v[q][r];  // canonical row R j + r, parked
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    stage_inv_rot(tiles[q], tw);
    {  // last inverse stage (span NJ; in place per item), then the tile leaves by TMA
      double2 v[NH][R];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int j = j0 + h * (T / 8);
#pragma unroll
        for (int r = 0; r < R; ++r) v[h][r] = tiles[q][tidx(j + r * NJ, c)];
#pragma unroll
        for (int r = 1; r < R; ++r) v[h][r] = cmul(v[h][r], cconj(tw[r * j]));
        dft_reg<R, true>(v[h]);
#pragma unroll
        for (int r = 0; r < R; ++r) tiles[q][tidx(j + r * NJ, c)] = v[h][r];
      }
    }
    fence_async();  // this thread's shared-memory writes -> visible to the async proxy
    __syncthreads();
    if (t == 0) {
      const unsigned src = m.tiles + q * kCompBytes;
      tma_store(m.spec, 2 * y0, 0, kx, m.lc0 + q, src);
      tma_store(m.spec, 2 * y0, L / 2, kx, m.lc0 + q, src + kCompBytes / 2);
      bulk_commit();
      if (q >= 1 && next >= 0) {  // the store of buffer q - 1 has read its tile: reload it
        bulk_wait_read<1>();
        load_comp(m, a, q - 1, next);
      }
    }
  }
  return part;
}
}  // namespace g5t

template <int MODE>
__global__ void __launch_bounds__(g5t::T, 1) gpass512e_tma_kernel(Ctx cx, const __grid_constant__ CUtensorMap tm_spec,
                                                                 const __grid_constant__ CUtensorMap tm_sym) {
  using namespace g5t;
  const Geo& g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ __align__(1024) double2 smem[];
  double2* tw = smem + NC * 8 * L;
  __shared__ double red_sh[32];
  __shared__ __align__(8) unsigned long long mbar[NC];
  for (int i = threadIdx.x; i < L; i += T) tw[i] = cx.tw.z[i];
  Args a;
  a.spec = cx.spec + (long long)load * g.c * g.nspec;
  a.gtab = cx.gtab;
  a.nspec = g.nspec;
  a.N2 = g.N2;
  a.N3 = g.N3;
  a.M = g.M;
  a.ntile_y = g.N2 >> 3;
  Tma m;
  m.spec = &tm_spec;
  m.sym = &tm_sym;
  m.tiles = sm_addr(smem);
  m.mbar = sm_addr(mbar);
  m.lc0 = load * g.c;
  const int ntiles = g.H1 * a.ntile_y;
  int tile = blockIdx.x;
  if (threadIdx.x == 0) {
    if (m.tiles & 1023u) __trap();  // SWIZZLE_128B needs the 1024-byte aligned tile base tidx assumes
#pragma unroll
    for (int q = 0; q < NC; ++q) mbar_init(m.mbar + 8 * q, 1);
    fence_async();
    if (tile < ntiles) {
#pragma unroll
      for (int q = 0; q < NC; ++q) load_comp(m, a, q, tile);
    }
  }
  __syncthreads();
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    const int next = tile + gridDim.x;
    const double part = g5t::tile_pass(a, m, tile, next < ntiles ? next : -1, it);
    partial_write<false>(cx, RED_GAMMA, load, tile, part, red_sh);
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

namespace g5 = g5e;

template <int MODE>
__global__ void __launch_bounds__(g5::T, 8 / g5::W) gpass512e_kernel(Ctx cx) {
  using namespace g5;
  const Geo& g = cx.g;
  const int load = blockIdx.y;
  if (MODE == CG && !cx.st[load].active) return;
  extern __shared__ double2 smem[];
  double2* tw = smem + NC * W * L;
  __shared__ double red_sh[32];
  for (int i = threadIdx.x; i < L; i += T) tw[i] = cx.tw.z[i];
  Args a;
  a.spec = cx.spec + (long long)load * g.c * g.nspec;
  a.gtab = cx.gtab;
  a.nspec = g.nspec;
  a.N2 = g.N2;
  a.N3 = g.N3;
  a.M = g.M;
  a.ntile_y = g.N2 / W;
  const int ntiles = g.H1 * a.ntile_y;
  int tile = blockIdx.x;
  if (tile < ntiles) {
    const long long b0 = tile_off(a, tile);
#pragma unroll
    for (int q = 0; q < NC; ++q) g5e::issue_t<T>(a, smem + q * W * L, q, b0);
  }
  for (; tile < ntiles; tile += gridDim.x) {
    const int next = tile + gridDim.x;
    const double part = g5::tile_pass(a, tile, next < ntiles ? next : -1);
    partial_write<false>(cx, RED_GAMMA, load, tile, part, red_sh);
  }
}

int gpass512e_nblk(const Geo& g) { return g.H1 * (g.N2 / g5e::W); }

bool gpass512e_supported(const Geo& g) {
  return UNO_G512E_PERSIST && g.dim == 3 && !g.dirz && !g.zpad && g.c == 3 && g.N3 == 512 && g.N2 % g5e::W == 0 &&
         (g5e::W == 8 || g.N2 == 512);  // W = 8: same tiles and gamma partial layout as gpass_z_kernel<512, 3>
}

#ifndef UNO_G5E_TMA
#define UNO_G5E_TMA 1  // 0: the cp.async version (A/B builds)
#endif
typedef CUresult (*TmEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmEncodeFn tm_encode_fn() {
  static TmEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (TmEncodeFn)p;
  }();
  return fn;
}
// 4D map over doubles: [n3][H1][N3][inner] with a box of `box0` doubles x 256 rows
static bool tm_make(CUtensorMap* tm, void* base, long long inner, int N3, int H1, long long n3, long long nspec_elems,
                    int elem_per_bin, int box0, bool swizzle) {
  TmEncodeFn enc = tm_encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)N3, (cuuint64_t)H1, (cuuint64_t)n3};
  const cuuint64_t strides[3] = {(cuuint64_t)inner * 8, (cuuint64_t)inner * 8 * N3,
                                 (cuuint64_t)nspec_elems * elem_per_bin * 8};
  const cuuint32_t box[4] = {(cuuint32_t)box0, 256, 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_gpass512e(const Ctx& cx, int mode, cudaStream_t s) {
  const Geo& g = cx.g;
  const int ntiles = gpass512e_nblk(g);
  const int ctas = kG512ePersistCTAs * (8 / g5e::W);
  const dim3 grid((unsigned)(ntiles < ctas ? ntiles : ctas), g.nrhs);
  constexpr int sm = (3 * g5e::W * 512 + 512) * (int)sizeof(double2);
#if UNO_G5E_TMA && UNO_G5E_W == 8
  CUtensorMap tm_spec, tm_sym;
  if (tm_make(&tm_spec, cx.spec, 2LL * g.N2, g.N3, g.H1, (long long)g.nrhs * g.c, g.nspec, 2, 16, true) &&
      tm_make(&tm_sym, const_cast<double*>(cx.gtab), g.N2, g.N3, g.H1, 6, g.nspec, 1, 8, false)) {
    auto go = [&](auto k) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm + 1024);
      k<<<grid, g5t::T, sm, s>>>(cx, tm_spec, tm_sym);
      return 1;
    };
    return mode == CG ? go(gpass512e_tma_kernel<CG>) : go(gpass512e_tma_kernel<STANDALONE>);
  }
#endif
  auto go = [&](auto k) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);  // per device: set on every launch
    k<<<grid, g5::T, sm, s>>>(cx);
    return 1;
  };
  return mode == CG ? go(gpass512e_kernel<CG>) : go(gpass512e_kernel<STANDALONE>);
}

}  // namespace uno
