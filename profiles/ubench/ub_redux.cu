#include <cstdint>
#include <cstdio>
__global__ void k(uint32_t* g, long long* res, int n) {
  uint32_t lane = threadIdx.x, x = g[lane];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __reduce_min_sync(0xffffffffu, x + lane) ;
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { unsigned b = __ballot_sync(0xffffffffu, (x + lane) & 1); x = __shfl_sync(0xffffffffu, x + 1, __ffs(b | 0x80000000u) - 1); }
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x + 1, 3);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) { unsigned b = __ballot_sync(0xffffffffu, (x + lane) & 1); x += __ffs(b | 0x80000000u); }
  long long t4 = clock64();
  if (lane == 0) { res[0] = (t1 - t0) / n; res[1] = (t2 - t1) / n; res[2] = (t3 - t2) / n; res[3] = (t4 - t3) / n; }
  g[lane] = x;
}
int main() { uint32_t* g; long long* r; cudaMalloc(&g, 128); cudaMalloc(&r, 64); cudaMemset(g, 0, 128);
  k<<<1,32>>>(g, r, 100); k<<<1,32>>>(g, r, 4000); long long h[4]; cudaMemcpy(h, r, 32, cudaMemcpyDeviceToHost);
  printf("redux.min chain %lld\nballot+ffs+shfl chain %lld\nshfl chain %lld\nballot+ffs chain %lld\n", h[0], h[1], h[2], h[3]); }
