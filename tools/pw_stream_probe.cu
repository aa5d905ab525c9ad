// Probe: what the memory system delivers for the PatchWeighted sweep's read pattern, with no arithmetic.
//   A  planar layout [k][row][col] read in the sweep's tiling (CTA = 8 rows x 128 columns, 24 x 16-byte loads per thread)
//   B  tiled layout  [col block][row][k][128 columns]: the same CTA reads one contiguous 96 KB piece
//   C  the same bytes as one flat stream (grid-stride 16-byte loads)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pw_stream_probe tools/pw_stream_probe.cu && /tmp/pw_stream_probe [H W]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
constexpr int NP = 24;
template <int LAYOUT, int MINB>
__global__ void __launch_bounds__(256, MINB) k_read(const float* __restrict__ w, float* out, int H, int W) {
  const int lane = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int i = blockIdx.y * 8 + r, jb = blockIdx.x, j = jb * 128 + 4 * lane;
  const long long N = (long long)H * W;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    long long o;
    if (LAYOUT == 0) o = (long long)k * N + (long long)i * W + j;
    else o = (((long long)jb * H + i) * NP + k) * 128 + 4 * lane;
    const float4 v = __ldg(reinterpret_cast<const float4*>(w + o));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.678f) out[0] = acc;
}
__global__ void __launch_bounds__(256) k_flat(const float4* __restrict__ w, float* out, long long n4) {
  float acc = 0.f;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += gridDim.x * 256LL) {
    const float4 v = __ldg(w + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.678f) out[0] = acc;
}
template <class F>
static float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}
int main(int argc, char** argv) {
  const int H = argc > 2 ? atoi(argv[1]) : 8192, W = argc > 2 ? atoi(argv[2]) : 8192;
  const long long n = (long long)NP * H * W;
  float *w, *out;
  cudaMalloc(&w, n * 4); cudaMalloc(&out, 4);
  cudaMemset(w, 0, n * 4);
  dim3 grid(W / 128, H / 8);
  const double gb = n * 4 / 1e9;
  float t;
  t = timeit([&] { k_read<0, 5><<<grid, 256>>>(w, out, H, W); }); printf("planar  5/SM %8.3f ms %7.1f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { k_read<0, 8><<<grid, 256>>>(w, out, H, W); }); printf("planar  8/SM %8.3f ms %7.1f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { k_read<1, 5><<<grid, 256>>>(w, out, H, W); }); printf("tiled   5/SM %8.3f ms %7.1f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { k_read<1, 8><<<grid, 256>>>(w, out, H, W); }); printf("tiled   8/SM %8.3f ms %7.1f GB/s\n", t, gb / t * 1e3);
  t = timeit([&] { k_flat<<<148 * 8, 256>>>(reinterpret_cast<const float4*>(w), out, n / 4); }); printf("flat         %8.3f ms %7.1f GB/s\n", t, gb / t * 1e3);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
