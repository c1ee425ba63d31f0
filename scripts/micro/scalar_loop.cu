// Cycles per request of the scalar walker's dense per-request loop (chunk.cu
// scalar_candidate: whole component state in every lane's registers, every
// group evaluated, one-hot argmin tree, predicated commit) for NG groups of S
// stages, one warp, a staged 32-request tile reused.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scalar_loop scalar_loop.cu
#include <cstdio>
#include <cstdint>
struct alignas(16) Req { unsigned ar, lim, tl, d[4], hm; int m, pad[3]; };

template <int S, int NG>
__global__ void loop(const Req* __restrict__ g, int iters, unsigned* out, long long* cyc, int id) {
  constexpr int R = NG * S;
  __shared__ Req tq[32];
  const int lane = threadIdx.x;
  tq[lane] = g[lane];
  __syncwarp();
  unsigned v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = r * 13u;
  unsigned good = 0, base = 0;
  unsigned long long sum = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int jj = 0; jj < 32; ++jj) {
      Req q = tq[jj];
      q.ar += base;
      q.lim += base;
      unsigned d[S];
#pragma unroll
      for (int k = 0; k < S; ++k) d[k] = q.d[k & 3];
      unsigned y[R], val[NG], oh[NG];
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        unsigned x = q.ar;
#pragma unroll
        for (int k = 0; k < S; ++k) {
          x = max(x, v[i * S + k]) + d[k];
          y[i * S + k] = x;
        }
        val[i] = ((q.hm >> i) & 1u) ? x : 0xFFFFFFFFu;
        oh[i] = 1u << i;
      }
#pragma unroll
      for (int st = 1; st < NG; st <<= 1)
#pragma unroll
        for (int i = 0; i + st < NG; i += 2 * st) {
          const bool p = val[i + st] < val[i];
          val[i] = p ? val[i + st] : val[i];
          oh[i] = p ? oh[i + st] : oh[i];
        }
      const bool acc = val[0] <= q.lim;
      const unsigned win = acc ? oh[0] : 0u;
#pragma unroll
      for (int i = 0; i < NG; ++i)
#pragma unroll
        for (int k = 0; k < S; ++k) v[i * S + k] = (win & (1u << i)) ? y[i * S + k] : v[i * S + k];
      good += acc;
      sum += acc ? (unsigned long long)(val[0] - q.ar + q.tl) : 0ull;
    }
    base += 1000u;
  }
  const long long t1 = clock64();
  unsigned acc = good + (unsigned)sum;
#pragma unroll
  for (int r = 0; r < R; ++r) acc += v[r];
  out[lane] = acc;
  if (lane == 0) cyc[id] = t1 - t0;
}

int main() {
  Req h[32];
  for (int i = 0; i < 32; ++i) {
    h[i].ar = i * 30u; h[i].lim = i * 30u + 400u; h[i].tl = 5u;
    for (int k = 0; k < 4; ++k) h[i].d[k] = 6u + k + (i % 3);
    h[i].hm = 0x3u >> (i % 2); h[i].m = i;
  }
  Req* g; unsigned* out; long long* cyc;
  cudaMalloc(&g, sizeof(h)); cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&out, 128); cudaMallocManaged(&cyc, 64);
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    loop<1, 8><<<1, 32>>>(g, iters, out, cyc, 0);
    loop<2, 2><<<1, 32>>>(g, iters, out, cyc, 1);
    loop<4, 2><<<1, 32>>>(g, iters, out, cyc, 2);
    loop<4, 4><<<1, 32>>>(g, iters, out, cyc, 3);
    loop<1, 1><<<1, 32>>>(g, iters, out, cyc, 4);
    cudaDeviceSynchronize();
  }
  const char* names[] = {"S=1 NG=8", "S=2 NG=2", "S=4 NG=2", "S=4 NG=4", "S=1 NG=1"};
  for (int k = 0; k < 5; ++k) printf("%-10s %.1f cycles/request\n", names[k], (double)cyc[k] / (iters * 32.0));
  return 0;
}
