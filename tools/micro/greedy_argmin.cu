// Microbenchmark: cycles per argmin round of a single warp over n shared-memory entries,
// with the other warps of a 1024-thread CTA parked at a barrier (as in k_reclaim) or absent.
#include <cstdio>
#include <cstdint>
__global__ void k(int n, int rounds, int park, long long* out) {
  __shared__ int64_t marg[2048];
  __shared__ int hid[2048];
  __shared__ unsigned char taken[2048];
  for (int i = threadIdx.x; i < n; i += blockDim.x) { marg[i] = (i * 7919) % 1000; hid[i] = i; taken[i] = 0; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    long long c0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      int64_t bm = 0; int bid = 0, bidx = -1;
#pragma unroll 4
      for (int i = lane; i < n; i += 32) {
        const int64_t m = marg[i]; const int id = hid[i];
        const bool better = !taken[i] && (bidx < 0 || m < bm || (m == bm && id < bid));
        bm = better ? m : bm; bid = better ? id : bid; bidx = better ? i : bidx;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t om = __shfl_xor_sync(~0u, bm, o);
        const int oid = __shfl_xor_sync(~0u, bid, o);
        const int oidx = __shfl_xor_sync(~0u, bidx, o);
        const bool better = oidx >= 0 && (bidx < 0 || om < bm || (om == bm && oid < bid));
        bm = better ? om : bm; bid = better ? oid : bid; bidx = better ? oidx : bidx;
      }
      if (lane == 0) { taken[bidx] = 1; atomicAdd((unsigned long long*)&marg[(bidx + 1) % n], 1ull); }
      __syncwarp();
    }
    long long c1 = clock64();
    if (lane == 0) out[0] = c1 - c0;
  }
  if (park) __syncthreads();
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  for (int park = 0; park < 2; ++park)
    for (int threads : {32, 1024}) {
      k<<<1, threads>>>(921, 36, park, d); cudaDeviceSynchronize();
      k<<<1, threads>>>(921, 36, park, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("threads=%d park=%d cycles/round=%lld err=%s\n", threads, park, h / 36, cudaGetErrorString(cudaGetLastError()));
    }
}
