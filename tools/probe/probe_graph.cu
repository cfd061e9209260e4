// Probe: CUDA graph conditional WHILE node driven by a device flag, and two
// streams ping-ponging through a device mailbox with release/acquire.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ int ld_acq(const int* p) { int v; asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }

// producer: bump counter, set loop condition while counter < n
__global__ void prod_step(int* mb, int n, cudaGraphConditionalHandle h) {
  int c = mb[0];
  // wait until consumer has caught up (ping-pong)
  while (ld_acq(&mb[1]) < c) { __nanosleep(100); }
  st_rel(&mb[0], c + 1);
  cudaGraphSetConditional(h, (c + 1) < n ? 1 : 0);
}
__global__ void cons_step(int* mb, int n, cudaGraphConditionalHandle h) {
  int c = mb[1];
  while (ld_acq(&mb[0]) <= c) { __nanosleep(100); }
  st_rel(&mb[1], c + 1);
  cudaGraphSetConditional(h, (c + 1) < n ? 1 : 0);
}

static int build_loop(cudaGraphExec_t* exec, void (*k)(int*, int, cudaGraphConditionalHandle), int* mb, int n) {
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  // capture the body via stream capture into the body graph
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  k<<<1, 32, 0, s>>>(mb, n, h);
  CK(cudaStreamEndCapture(s, &body));
  CK(cudaGraphInstantiate(exec, g, 0));
  return 0;
}


__global__ void tiny(float* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0f; }
__global__ void tiny_pdl(float* x) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0f;
  asm volatile("griddepcontrol.launch_dependents;");
}
static int chain(bool pdl, int blocks) {
  float* x; CK(cudaMalloc(&x, 4));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < 200; ++i) {
    if (!pdl) { tiny<<<blocks, 128, 0, s>>>(x); }
    else {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(128); cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, tiny_pdl, x));
    }
  }
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaEventRecord(e0, s)); for (int r = 0; r < 10; ++r) CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("graph chain pdl=%d blocks=%d: %.3f us per kernel\n", (int)pdl, blocks, 1000.0f * ms / 2000.0f);
  return 0;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s sm_%d%d SMs=%d l2=%d MB smemOptin=%zu\n", p.name, p.major, p.minor, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin);
  int* mb; CK(cudaMalloc(&mb, 64)); CK(cudaMemset(mb, 0, 64));
  const int n = 10000;
  cudaGraphExec_t ep, ec;
  if (build_loop(&ep, prod_step, mb, n)) return 1;
  if (build_loop(&ec, cons_step, mb, n)) return 1;
  cudaStream_t s1, s2; CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaEventRecord(e0, s1));
  CK(cudaGraphLaunch(ep, s1));
  CK(cudaGraphLaunch(ec, s2));
  CK(cudaStreamSynchronize(s1)); CK(cudaStreamSynchronize(s2));
  CK(cudaEventRecord(e1, s1)); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int h[2]; CK(cudaMemcpy(h, mb, 8, cudaMemcpyDeviceToHost));
  printf("pingpong prod=%d cons=%d in %.3f ms => %.2f us per round trip\n", h[0], h[1], ms, 1000.0 * ms / n);
  chain(false, 1); chain(true, 1); chain(false, 296); chain(true, 296);
  return 0;
}
