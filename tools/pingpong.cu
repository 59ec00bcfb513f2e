// Flag round trip between two GPUs over NVLink (one process, peer access):
// thread 0 of one CTA on each GPU; GPU A stores i into B's memory, B polls
// its own memory for it and answers into A's memory. Compares the polling
// load (ld.acquire.sys every iteration / ld.relaxed.sys then one acquire /
// ld.volatile) and the publishing store (st.release.sys / st.relaxed.sys),
// i.e. the latency each handshake of the collectives' flag protocol costs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/pingpong tools/pingpong.cu
//   tools/pingpong [devA devB]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

__device__ __forceinline__ unsigned long long poll(const unsigned long long *p, int mode) {
  unsigned long long v;
  if (mode == 0) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else if (mode == 1) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void publish(unsigned long long *p, unsigned long long v, int mode) {
  if (mode == 0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// me: my own flag word (polled); other: the peer's flag word (written)
__global__ void k_pingpong(unsigned long long *me, unsigned long long *other, int first, int iters, int pmode,
                           int smode, unsigned long long base, long long *ns) {
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  for (int i = 1; i <= iters; ++i) {
    const unsigned long long v = base + i;
    if (first) {
      publish(other, v, smode);
      while (poll(me, pmode) < v) {
      }
    } else {
      while (poll(me, pmode) < v) {
      }
      publish(other, v, smode);
    }
    if (pmode == 1) {  // the acquire that the relaxed polling defers
      unsigned long long w;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(me) : "memory");
      if (w == ~0ull) *ns = -1;
    }
  }
  unsigned long long t_end;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
  *ns = (long long)(t_end - t_start);
  (void)t0;
}

int main(int argc, char **argv) {
  const int a = argc > 2 ? atoi(argv[1]) : 0, b = argc > 2 ? atoi(argv[2]) : 1;
  unsigned long long *fa, *fb;
  long long *na, *nb;
  CK(cudaSetDevice(a));
  CK(cudaDeviceEnablePeerAccess(b, 0));
  CK(cudaMalloc(&fa, 64));
  CK(cudaMemset(fa, 0, 64));
  CK(cudaMallocManaged(&na, 8));
  CK(cudaSetDevice(b));
  CK(cudaDeviceEnablePeerAccess(a, 0));
  CK(cudaMalloc(&fb, 64));
  CK(cudaMemset(fb, 0, 64));
  CK(cudaMallocManaged(&nb, 8));
  cudaStream_t sa, sb;
  CK(cudaSetDevice(a));
  CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  CK(cudaSetDevice(b));
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  const char *pm[] = {"ld.acquire.sys", "ld.relaxed.sys + acquire", "ld.volatile"};
  const char *sm[] = {"st.release.sys", "st.relaxed.sys"};
  unsigned long long base = 0;
  const int iters = 2000;
  printf("GPU %d <-> GPU %d flag round trips (%d per run)\n", a, b, iters);
  for (int pmode = 0; pmode < 3; ++pmode)
    for (int smode = 0; smode < 2; ++smode) {
      CK(cudaSetDevice(b));
      k_pingpong<<<1, 32, 0, sb>>>(fb, fa, 0, iters, pmode, smode, base, nb);
      CK(cudaSetDevice(a));
      k_pingpong<<<1, 32, 0, sa>>>(fa, fb, 1, iters, pmode, smode, base, na);
      CK(cudaStreamSynchronize(sa));
      CK(cudaSetDevice(b));
      CK(cudaStreamSynchronize(sb));
      base += iters;
      printf("  poll %-26s publish %-15s  %6.3f us per round trip\n", pm[pmode], sm[smode], *na / 1e3 / iters);
    }
  return 0;
}
