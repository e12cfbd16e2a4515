// Probe (not product code): cost of a chain of dependent kernel launches in a
// CUDA graph on B200, empty vs. with a few dependent global loads per CTA.
#include <cstdio>
#include <cuda_runtime.h>
struct Args { int* p[8]; };
__global__ void k_empty(const Args* a, int s) {}
__global__ void k_chain(const Args* a, int s) {  // 4 dependent loads, like the phase kernels' prologue
  const Args& A = *a;
  int* q = A.p[s & 7];
  int v = *(volatile int*)q;
  int w = *(volatile int*)(A.p[(v + 1) & 7]);
  int x = *(volatile int*)(A.p[(w + 2) & 7]);
  if (x == 12345 && threadIdx.x == 0) A.p[0][1] = s;
}
int main() {
  Args h; int* buf; cudaMalloc(&buf, 1 << 20); cudaMemset(buf, 0, 1 << 20);
  for (int i = 0; i < 8; ++i) h.p[i] = buf + i * 1024;
  Args* d; cudaMalloc(&d, sizeof(Args)); cudaMemcpy(d, &h, sizeof(Args), cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int variant = 0; variant < 4; ++variant) {
    int grid = (variant & 1) ? 148 : 740;
    cudaGraph_t g; cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 2200; ++i) {
      if (variant < 2) k_empty<<<grid, 256, 0, st>>>(d, i); else k_chain<<<grid, 256, 0, st>>>(d, i);
    }
    cudaStreamEndCapture(st, &g); cudaGraphExec_t e; cudaGraphInstantiate(&e, g, 0);
    cudaGraphLaunch(e, st); cudaStreamSynchronize(st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, st); cudaGraphLaunch(e, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s grid %d: %.3f ms for 2200 launches = %.2f us each\n", variant < 2 ? "empty" : "chain4", grid, ms, ms * 1e3 / 2200);
  }
  return 0;
}
