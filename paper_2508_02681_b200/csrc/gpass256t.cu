// gpass256t.cu — thermal G pass at N3 = 256 (config 3, the headline): z FFT -> s_hat = G_hat r_hat
// and the Parseval partial of gamma_1 (Eq 46/49) -> inverse z FFT (Alg 2 l.4-7), in place
// on the half spectrum [load][kx][z][y], as a TMA-streamed persistent kernel.
//
// Work unit = (tile, load): 8 y columns x 256 z of one kx plane of one load case (32 KB; rows of
// 128 bytes at stride N2 * 16).  A CTA (128 threads, two per SM) walks its units — load fastest, so
// the symbol of a tile is fetched once and stays in registers for the tile's loads — through a ring
// of three 32 KB buffers: cp.async.bulk.tensor loads complete on one mbarrier per buffer, the
// result leaves by a bulk tensor store, and the buffer of unit u - 1 is reloaded for unit u + 2 once
// that store has read it (cp.async.bulk.wait_group.read).  The compute threads issue no global
// loads or stores for the tiles, and memory latency is covered by the ring instead of by occupancy
// (the register-direct gpass256_kernel keeps three CTAs per SM waiting on their own loads).
// CU_TENSOR_MAP_SWIZZLE_128B is fft.cuh's tidx swizzle (16-byte chunk c of row j at c ^ (j & 7)).
//
// 256 = 16 . 16, one radix-16 butterfly per thread and pass, three passes per unit:
//   P1  first forward stage (span 1): rows j + 16 r -> rows 16 j + r                  (barrier inside)
//   MID last forward stage (span 16) on rows j + 16 r -> multiply the bins j + 16 r by G_hat ->
//       first inverse stage (span 1), outputs (canonical rows 16 j + r) parked in the item's own rows
//       j + 16 r: no other item's data is touched, no barrier inside
//   P3  last inverse stage (span 16) reading canonical rows j + 16 r through the parking
//       permutation (= rows 16 j + r), writing rows j + 16 r                          (barrier inside)
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"
#include "dev_common.cuh"

namespace uno {

#ifndef UNO_SERP
#define UNO_SERP 1  // reversed tile order (see ypass256_kernel); 0: A/B
#endif
#ifndef UNO_G256T_NB
#define UNO_G256T_NB 2  // ring buffers per CTA: 2 (three CTAs per SM, 168 registers) or 3 (two CTAs per SM)
#endif
#ifndef UNO_G256T
#define UNO_G256T 1  // 0: the register-direct gpass256_kernel (A/B builds)
#endif

namespace g2t {
constexpr int L = 256, T = 128, R = 16, NJ = L / R, NB = UNO_G256T_NB;  // NB ring buffers
constexpr unsigned kTileBytes = 8 * L * 16;
constexpr int kCtasPerSm = NB == 1 ? 4 : (NB == 2 ? 3 : 2), kCtas = 148 * kCtasPerSm;
static_assert(NJ * kTile == T && T == 128, "one butterfly per thread in every pass; four warps (gamma partial)");

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
      "G2T_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra G2T_DONE;\n"
      "bra G2T_WAIT;\n"
      "G2T_DONE:\n"
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

struct Args {
  const CUtensorMap* spec;  // doubles [load][kx][z][2 y], box 16 x 256, SWIZZLE_128B
  const CUtensorMap* sym;   // doubles [1][kx][z][y], box 8 x 256 (L2 prefetch only)
  const double* gtab;
  unsigned tiles, mbar;     // shared-memory addresses of buffer 0 and of the NB mbarriers
  int N2, N3, M, ntile_y, ntiles;
  int nact;                 // active load cases
  int act[kMaxRhs];         // their indices
};

// unit u of this CTA -> (tile, load)
__device__ __forceinline__ void unit_of(const Args& a, long long u, int& tile, int& load) {
  const long long gt = u / a.nact;
  tile = (int)(blockIdx.x + gt * gridDim.x);
#if UNO_SERP
  tile = a.ntiles - 1 - tile;  // last k_x planes first: they are what the forward y pass left in L2
#endif
  load = a.act[(int)(u - gt * a.nact)];
}
// thread 0: load unit (tile, load) into ring buffer b; the first load of a tile also pulls the
// tile's symbol rows into L2
__device__ __forceinline__ void load_unit(const Args& a, int b, int tile, int load, bool first_of_tile) {
  const int kx = tile / a.ntile_y, y0 = (tile - kx * a.ntile_y) * 8;
  const unsigned mb = a.mbar + 8 * b;
  mbar_expect_tx(mb, kTileBytes);
  tma_load(a.tiles + b * kTileBytes, a.spec, 2 * y0, 0, kx, load, mb);
  if (first_of_tile) tma_prefetch(a.sym, y0, 0, kx, 0);
}
}  // namespace g2t

template <int MODE>
__global__ void __launch_bounds__(g2t::T, g2t::kCtasPerSm) gpass256t_kernel(Ctx cx, const __grid_constant__ CUtensorMap tm_spec,
                                                                           const __grid_constant__ CUtensorMap tm_sym) {
  using namespace g2t;
  const Geo& g = cx.g;
  extern __shared__ __align__(1024) double2 smem[];
  double2* tw = smem + NB * 8 * L;
  __shared__ double red_sh[32];
  __shared__ __align__(8) unsigned long long mbar[NB];
  const int t = threadIdx.x, c = t & 7, j = t >> 3;
  Args a;
  a.spec = &tm_spec;
  a.sym = &tm_sym;
  a.gtab = cx.gtab;
  a.tiles = sm_addr(smem);
  a.mbar = sm_addr(mbar);
  a.N2 = g.N2;
  a.N3 = g.N3;
  a.M = g.M;
  a.ntile_y = g.N2 >> 3;
  a.nact = 0;
#pragma unroll
  for (int l = 0; l < kMaxRhs; ++l) {
    a.act[l] = 0;
    if (l < g.nrhs && (MODE != CG || cx.st[l].active)) a.act[a.nact++] = l;
  }
  if (a.nact == 0) return;
  const int ntiles = g.H1 * a.ntile_y;
  a.ntiles = ntiles;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const long long nunits = (long long)my_tiles * a.nact;
  for (int i = t; i < L; i += T) tw[i] = cx.tw.z[i];
  if (t == 0) {
    if (a.tiles & 1023u) __trap();  // SWIZZLE_128B needs the 1024-byte aligned buffers tidx assumes
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(a.mbar + 8 * b, 1);
    fence_async();
    for (int u = 0; u < NB && u < nunits; ++u) {
      int tile, load;
      unit_of(a, u, tile, load);
      load_unit(a, u, tile, load, u % a.nact == 0);
    }
  }
  __syncthreads();
  double gsym[R];  // symbol of the bins j + 16 r of column c, kept for the loads of a tile
  int sym_tile = -1;
#pragma unroll 1
  for (long long u = 0; u < nunits; ++u) {
    int tile, load;
    unit_of(a, u, tile, load);
    const int b = (int)(u % NB);
    double2* s = smem + b * 8 * L;
    const int kx = tile / a.ntile_y, y0 = (tile - kx * a.ntile_y) * 8;
    if (tile != sym_tile) {  // issued before the wait so the loads overlap it
      const double* gp = a.gtab + (long long)kx * a.N3 * a.N2 + y0 + c;
#pragma unroll
      for (int r = 0; r < R; ++r) gsym[r] = __ldg(gp + (long long)(j + r * NJ) * a.N2);
      sym_tile = tile;
    }
    mbar_wait(a.mbar + 8 * b, (unsigned)((u / NB) & 1));
    double2 v[R];
    // P1: first forward stage (span 1)
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[tidx(j + r * NJ, c)];
    Dft<R>::run(v);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) s[tidx(j * R + r, c)] = v[r];
    __syncthreads();
    if (NB == 2 && t == 0 && u >= 1 && u + 1 < nunits) {  // two buffers: the other one (unit u - 1) has been
      bulk_wait_read<0>();                                 // stored a third of a unit ago: reload it for unit u + 1
      int tile2, load2;
      unit_of(a, u + 1, tile2, load2);
      load_unit(a, (int)((u + 1) % NB), tile2, load2, (u + 1) % a.nact == 0);
    }
    // MID: last forward stage (span 16), symbol multiply, first inverse stage (span 1), own rows
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[tidx(j + r * NJ, c)];
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * j]);
    Dft<R>::run(v);
    const double w = parseval_w(kx, a.M);
    double part = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double gv = gsym[r];
      part += w * gv * fma(v[r].x, v[r].x, v[r].y * v[r].y);
      v[r] = make_double2(gv * v[r].x, gv * v[r].y);
    }
    dft_reg_inv_inline<R>(v);
#pragma unroll
    for (int r = 0; r < R; ++r) s[tidx(j + r * NJ, c)] = v[r];  // canonical row 16 j + r, parked
    // gamma partial of the unit (same tree and order as block_reduce), riding on the barrier the
    // stages need anyway instead of two barriers of its own
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if ((t & 31) == 0) red_sh[t >> 5] = part;
    __syncthreads();
    if (t == 0) red_partials(cx.sc, RED_GAMMA, load)[tile] = ((red_sh[0] + red_sh[1]) + red_sh[2]) + red_sh[3];
    // P3: last inverse stage (span 16): canonical rows j + 16 r are parked at rows 16 j + r
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[tidx(j * R + r, c)];
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], cconj(tw[r * j]));
    dft_reg<R, true>(v);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) s[tidx(j + r * NJ, c)] = v[r];
    fence_async();  // this thread's shared-memory writes -> visible to the async proxy
    __syncthreads();
    if (t == 0) {
      tma_store(a.spec, 2 * y0, 0, kx, load, a.tiles + b * kTileBytes);
      bulk_commit();
      if (NB == 1 && u + 1 < nunits) {  // single buffer (four CTAs per SM cover each other's waits)
        bulk_wait_read<0>();
        int tile2, load2;
        unit_of(a, u + 1, tile2, load2);
        load_unit(a, 0, tile2, load2, (u + 1) % a.nact == 0);
      }
      if (NB == 3 && u >= 1 && u + 2 < nunits) {  // the store of unit u - 1 has read its buffer: reload it for unit u + 2
        bulk_wait_read<1>();
        int tile2, load2;
        unit_of(a, u + 2, tile2, load2);
        load_unit(a, (int)((u + 2) % NB), tile2, load2, (u + 2) % a.nact == 0);
      }
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

bool gpass256t_supported(const Geo& g) {
  return UNO_G256T && g.dim == 3 && !g.dirz && !g.zpad && g.c == 1 && g.N3 == 256 && g.N2 % 8 == 0 && g.N2 >= 8;
}

typedef CUresult (*TmEncodeFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmEncodeFn2 tm_encode_fn2() {
  static TmEncodeFn2 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (TmEncodeFn2)p;
  }();
  return fn;
}
static bool tm_make2(CUtensorMap* tm, void* base, long long inner, int N3, int H1, long long n3, long long outer_stride_bytes,
                     int box0, bool swizzle) {
  TmEncodeFn2 enc = tm_encode_fn2();
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)N3, (cuuint64_t)H1, (cuuint64_t)n3};
  const cuuint64_t strides[3] = {(cuuint64_t)inner * 8, (cuuint64_t)inner * 8 * N3, (cuuint64_t)outer_stride_bytes};
  const cuuint32_t box[4] = {(cuuint32_t)box0, 256, 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// returns 1 on launch, -1 if the tensor maps cannot be encoded (caller falls back to gpass256_kernel)
int launch_gpass256t(const Ctx& cx, int mode, cudaStream_t s) {
  using namespace g2t;
  const Geo& g = cx.g;
  CUtensorMap tm_spec, tm_sym;
  if (!tm_make2(&tm_spec, cx.spec, 2LL * g.N2, g.N3, g.H1, (long long)g.nrhs * g.c, g.nspec * 16, 16, true) ||
      !tm_make2(&tm_sym, const_cast<double*>(cx.gtab), g.N2, g.N3, g.H1, 1, g.nspec * 8, 8, false))
    return -1;
  const int ntiles = g.H1 * (g.N2 / 8);
  const dim3 grid((unsigned)(ntiles < kCtas ? ntiles : kCtas));
  constexpr int sm = (NB * 8 * L + L) * (int)sizeof(double2);
  auto go = [&](auto k) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);  // per device: set on every launch
    k<<<grid, T, sm, s>>>(cx, tm_spec, tm_sym);
    return 1;
  };
  return mode == CG ? go(gpass256t_kernel<CG>) : go(gpass256t_kernel<STANDALONE>);
}

}  // namespace uno
