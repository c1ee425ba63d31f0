// Cycles per request of the group-lane walker's per-request loop (S = 2, one
// warp, a 32-request staged tile reused): the dependent chain of
// chunk.cu glane_candidate, isolated from the tile staging and the trace.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o glane_loop glane_loop.cu
#include <cstdio>
#include <cstdint>
constexpr unsigned FULL = 0xFFFFFFFFu;
struct alignas(16) Req { unsigned ar, lim, d0, tl, d1, hm; int m, pad; };

template <int MODE>
__global__ void loop(const Req* __restrict__ g, int iters, unsigned* out, long long* cyc) {
  __shared__ Req tqs[32][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Req* tq = tqs[wid];
  tq[lane] = g[lane];
  __syncwarp();
  unsigned v0 = lane * 7u, v1 = lane * 11u, good = 0, base = 0;
  unsigned long long sum = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int jj = 0; jj < 32; ++jj) {
      Req q = tq[jj];
      q.ar += base;
      q.lim += base;
      unsigned x = max(q.ar, v0) + q.d0;
      const unsigned y0 = x;
      x = max(x, v1) + q.d1;
      const unsigned key = ((q.hm >> lane) & 1u) ? x : 0xFFFFFFFFu;
      unsigned mn, win;
      if (MODE == 0) {  // exact min, then the lowest lane among the minima
        mn = __reduce_min_sync(FULL, key);
        win = __reduce_min_sync(FULL, key == mn ? (unsigned)lane : 32u);
      } else {  // exact min and coarse key together
        mn = __reduce_min_sync(FULL, key);
        const unsigned cw = __reduce_min_sync(FULL, (key & ~31u) | (unsigned)lane);
        win = cw & 31u;
        if (__shfl_sync(FULL, key, win) != mn) win = __reduce_min_sync(FULL, key == mn ? (unsigned)lane : 32u);
      }
      const bool acc = mn <= q.lim;
      const bool take = acc && (unsigned)lane == win;
      v0 = take ? y0 : v0;
      v1 = take ? x : v1;
      good += acc;
      sum += acc ? (unsigned long long)(mn - q.ar + q.tl) : 0ull;
    }
    base += 1000u;
  }
  const long long t1 = clock64();
  out[threadIdx.x] = v0 + v1 + good + (unsigned)sum;
  if (threadIdx.x == 0) cyc[MODE] = t1 - t0;
}

int main() {
  Req h[32];
  for (int i = 0; i < 32; ++i) {
    h[i].ar = i * 30u; h[i].lim = i * 30u + 400u; h[i].d0 = 20u + (i % 3); h[i].d1 = 25u;
    h[i].tl = 5u; h[i].hm = 0x0Fu << (i % 4); h[i].m = i; h[i].pad = 0;
  }
  Req* g; unsigned* out; long long* cyc;
  cudaMalloc(&g, sizeof(h)); cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&out, 32 * 32 * 4); cudaMallocManaged(&cyc, 16);
  const int iters = 2000;
  // one walker warp alone, then 4 / 8 / 16 co-resident warps in one block
  // (one SM): does the warp-min unit serialise co-resident walkers?
  for (int nw : {1, 4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      loop<0><<<1, 32 * nw>>>(g, iters, out, cyc);
      loop<1><<<1, 32 * nw>>>(g, iters, out, cyc);
      cudaDeviceSynchronize();
    }
    printf("%2d warps/SM: two warp mins in sequence %.1f, exact + coarse %.1f cycles/request\n", nw,
           (double)cyc[0] / (iters * 32.0), (double)cyc[1] / (iters * 32.0));
  }
  return 0;
}
