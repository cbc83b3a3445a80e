// Probe: resident CTAs per SM of a 96-thread kernel against its dynamic shared memory size.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __maxnreg__(96) k(float* p) {
  extern __shared__ float s[];
  s[threadIdx.x] = p[threadIdx.x];
  __syncthreads();
  p[threadIdx.x] = s[(threadIdx.x + 1) % 96];
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  int last = -1;
  for (int smem = 32336; smem >= 32100; smem -= 8) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 96, smem);
    if (n != last) printf("smem %d -> %d CTAs/SM\n", smem, n);
    last = n;
  }
  return 0;
}
