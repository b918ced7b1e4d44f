// Strided-tile read-modify-write probe: the memory access pattern of the z (G) passes without any
// arithmetic.  A CTA owns a tile of R rows x W bytes (row r at base + r * S), loads all of it into
// registers, and writes it back in place — the pattern of gpass256 (R = 256, S = 528,384 B) and of
// the 512-point G passes (R = 512, S = 2,105,344 B).  Question: is the 512^3 z pass slow because
// of its kernels or because every row of a tile lies in a different 2 MB page?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stride_tile stride_tile.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__);        \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// T threads; W bytes per row (W/16 threads per row); R rows; per-thread R*W/16/T 16-byte vectors
template <int R, int W, int T>
__global__ void __launch_bounds__(T) rmw(double2* buf, long long S16, long long tiles_per_arr, long long arr16,
                                         long long blk_tiles, long long blk16, int W16tile) {
  constexpr int LW = W / 16, RPI = T / LW, NV = R / RPI;
  const long long t = blockIdx.x;
  const long long a = t / tiles_per_arr, u = t % tiles_per_arr;
  // blocked layouts: tile u lives in block u / blk_tiles at offset (u % blk_tiles) * W16tile
  double2* base = buf + a * arr16 + (u / blk_tiles) * blk16 + (u % blk_tiles) * W16tile;
  const int lx = threadIdx.x % LW, r0 = threadIdx.x / LW;
  double2 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = base[(long long)(r0 + i * RPI) * S16 + lx];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i].x += 1.0;
    base[(long long)(r0 + i * RPI) * S16 + lx] = v[i];
  }
}

template <int R, int W, int T>
static void run(const char* name, double2* buf, long long S, long long tiles_per_arr, int narr, long long arr_bytes,
                long long blk_tiles, long long blk_bytes) {
  const long long tiles = tiles_per_arr * narr;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 2; ++i)
    rmw<R, W, T><<<(unsigned)tiles, T>>>(buf, S / 16, tiles_per_arr, arr_bytes / 16, blk_tiles, blk_bytes / 16, W / 16);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i)
    rmw<R, W, T><<<(unsigned)tiles, T>>>(buf, S / 16, tiles_per_arr, arr_bytes / 16, blk_tiles, blk_bytes / 16, W / 16);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double bytes = 2.0 * tiles * R * W;
  printf("%-46s R=%d W=%d T=%d stride=%lld B: %.1f us  %.2f TB/s\n", name, R, W, T, S, 1e3 * ms / reps,
         bytes * reps / (ms * 1e-3) / 1e12);
}

int main() {
  const long long GB4 = 3ll * 512 * 512 * 257 * 16 + (64 << 20);
  double2* buf;
  CK(cudaMalloc(&buf, GB4));
  CK(cudaMemset(buf, 0, GB4));
  // 256^3 thermal, 3 loads: plane 256 x 129 bins
  {
    const long long S = 256ll * 129 * 16, arr = S * 256;
    run<256, 128, 256>("256^3 x3 z tiles (gpass256 pattern)", buf, S, 256 * 129 / 8, 3, arr, 1ll << 40, 0);
    run<256, 64, 256>("256^3 x3 z tiles, 4 columns", buf, S, 256 * 129 / 4, 3, arr, 1ll << 40, 0);
  }
  // 512^3 x 3 components: plane 512 x 257 bins
  {
    const long long S = 512ll * 257 * 16, arr = S * 512;
    run<512, 128, 256>("512^3 x3 z tiles (plane-major layout)", buf, S, 512 * 257 / 8, 3, arr, 1ll << 40, 0);
    run<512, 128, 512>("512^3 x3 z tiles (plane-major), 512 thr", buf, S, 512 * 257 / 8, 3, arr, 1ll << 40, 0);
    run<512, 64, 256>("512^3 x3 z tiles, 4 columns", buf, S, 512 * 257 / 4, 3, arr, 1ll << 40, 0);
    run<256, 128, 256>("512^3 x3 half columns (R=256 of 512)", buf, S, 512 * 257 / 8, 3, arr, 1ll << 40, 0);
    // blocked layout [yb][z][8 rows][257]: z stride 8*257*16, block = 512 * that
    const long long Sb = 8ll * 257 * 16, blk = Sb * 512;
    run<512, 128, 256>("512^3 x3 z tiles, y-blocked layout (B=8)", buf, Sb, 512 * 257 / 8, 3, arr, 257, blk);
    const long long Sb2 = 32ll * 257 * 16, blk2 = Sb2 * 512;
    run<512, 128, 256>("512^3 x3 z tiles, y-blocked layout (B=32)", buf, Sb2, 512 * 257 / 8, 3, arr, 257 * 4, blk2);
    // contiguous reference: same bytes, rows adjacent (S = W)
    run<512, 128, 256>("512^3 x3 contiguous tiles", buf, 128, 512 * 257 / 8, 3, arr, 1, 512ll * 128);
  }
  // y-pass pattern at 512: rows of one z plane, tile = 8 columns, stride 257*16
  {
    const long long S = 257ll * 16, pl = S * 512;
    // tile u of array a: plane p = u / 32, column tile u % 32 (257th bin ignored)
    run<512, 128, 256>("512^3 y tiles (row stride 4112 B)", buf, S, 512 * 3 * 32, 1, 0, 32, pl);
  }
  CK(cudaFree(buf));
  return 0;
}
