// Probe: device-side (CDP2) tail launch from a one-thread dispatcher kernel, sized from a
// device-resident count; checks that later host-stream work observes the child's writes.
// nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -O3 cdp_tail_probe.cu -lcudadevrt -o cdp_tail_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void child(int *out, int n, int tag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = tag + i;
}
__global__ void dispatch(const int *n_dev, int *out, int tag) {
  int n = *n_dev;
  if (n > 0) child<<<(n + 255) / 256, 256, 0, cudaStreamTailLaunch>>>(out, n, tag);
}
__global__ void check(const int *out, int n, int tag, int *bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && out[i] != tag + i) atomicAdd(bad, 1);
}
int main() {
  int *n_dev, *out, *bad;
  cudaMalloc(&n_dev, 4); cudaMalloc(&out, 4 << 22); cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 200; ++it) {
    int n = 1000 + it * 20000;
    cudaMemcpyAsync(n_dev, &n, 4, cudaMemcpyHostToDevice, st);
    if (it == 100) cudaEventRecord(a, st);
    dispatch<<<1, 1, 0, st>>>(n_dev, out, it);
    check<<<(n + 255) / 256, 256, 0, st>>>(out, n, it, bad);
    if (it == 100) cudaEventRecord(b, st);
  }
  int h = -1;
  cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\":\"cdp_tail\",\"err\":\"%s\",\"bad\":%d,\"dispatch_plus_check_us\":%.2f}\n",
         cudaGetErrorString(e), h, ms * 1e3);
  return 0;
}
