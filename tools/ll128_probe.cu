// LL128 feasibility probe: can a 128-byte line written
// by 8 lanes of one warp store instruction (7 x 16 B payload + 8 B payload +
// 8 B flag) be trusted as a unit over NVLink on B200, and what bandwidth does
// such a line protocol move? One process, two GPUs with peer access, both
// directions loaded at once (every collective loads both). Each round r, the
// sender on each GPU writes the whole region of lines into the peer's memory
// with tag r; the receiver polls every line until its flag says r, then checks
// all 120 payload bytes against round r (a "torn" line = flag new, payload
// old) and publishes one round-done word back; the sender waits for it before
// round r + 1. Not used by the library: the measurement that decides whether
// an LL128 protocol is worth building.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/ll128_probe tools/ll128_probe.cu
//   tools/ll128_probe [devA devB] [MiB per round] [rounds]
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

__device__ __forceinline__ unsigned long long payload(unsigned long long line, int j, unsigned long long r) {
  return (line * 0x9E3779B97F4A7C15ull) ^ ((unsigned long long)j << 56) ^ (r * 0xD1B54A32D192ED03ull);
}

__device__ __forceinline__ void st_v2(unsigned long long *p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_v2(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// One kernel per GPU per round: CTAs [0, C) send, CTAs [C, 2C) receive.
// lines: number of 128-byte lines per round; out: the peer's region (written),
// in: my region (polled). done_peer / done_me: round-done words.
__global__ void k_round(unsigned long long *out, const unsigned long long *in, long long lines, unsigned long long r,
                        unsigned long long *done_peer, const unsigned long long *done_me, int C,
                        unsigned long long *torn) {
  const int lane = threadIdx.x & 31, j = lane & 7;
  const long long warps_per_cta = blockDim.x / 32;
  if ((int)blockIdx.x < C) {  // sender: wait until the peer consumed round r - 1, then stream lines
    if (threadIdx.x == 0) {
      unsigned long long v;
      do {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(done_me) : "memory");
      } while (v + 1 < r);
    }
    __syncthreads();
    const long long w0 = (long long)blockIdx.x * warps_per_cta + threadIdx.x / 32;
    for (long long g = w0; g * 4 < lines; g += (long long)C * warps_per_cta) {
      const long long line = g * 4 + lane / 8;
      if (line >= lines) continue;
      unsigned long long *p = out + line * 16 + j * 2;
      if (j < 7) st_v2(p, payload(line, 2 * j, r), payload(line, 2 * j + 1, r));
      else st_v2(p, payload(line, 14, r), r);  // last 8 bytes: the flag
    }
  } else {  // receiver: poll my region until every line carries round r, check its payload
    const int b = blockIdx.x - C;
    unsigned long long bad = 0;
    const long long w0 = (long long)b * warps_per_cta + threadIdx.x / 32;
    for (long long g = w0; g * 4 < lines; g += (long long)C * warps_per_cta) {
      const long long line = g * 4 + lane / 8;
      const bool valid = line < lines;
      const unsigned long long *p = in + (valid ? line : 0) * 16 + j * 2;
      unsigned long long a, c;
      while (true) {
        ld_v2(p, a, c);
        const bool ready = !valid || j != 7 || c == r;
        if (__all_sync(0xffffffffu, ready)) break;
      }
      if (valid) {
        if (j < 7) bad += (a != payload(line, 2 * j, r)) || (c != payload(line, 2 * j + 1, r));
        else bad += a != payload(line, 14, r);
      }
    }
    if (bad) atomicAdd(torn, bad);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      // round done when every receiving CTA has finished: a local counter in `torn`[1]
      const unsigned long long old = atomicAdd(torn + 1, 1ull);
      if (old + 1 == (unsigned long long)C * r) {
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(done_peer), "l"(r) : "memory");
      }
    }
  }
}

int main(int argc, char **argv) {
  const int a = argc > 2 ? atoi(argv[1]) : 0, b = argc > 2 ? atoi(argv[2]) : 1;
  const long long mib = argc > 3 ? atoll(argv[3]) : 64;
  const int rounds = argc > 4 ? atoi(argv[4]) : 200;
  const long long lines = (mib << 20) / 128;
  const int C = 64;
  unsigned long long *reg[2], *done[2], *torn[2];
  const int dev[2] = {a, b};
  for (int i = 0; i < 2; ++i) {
    CK(cudaSetDevice(dev[i]));
    cudaError_t e = cudaDeviceEnablePeerAccess(dev[1 - i], 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
    cudaGetLastError();
    CK(cudaMalloc(&reg[i], lines * 128));
    CK(cudaMemset(reg[i], 0, lines * 128));
    CK(cudaMalloc(&done[i], 64));
    CK(cudaMemset(done[i], 0, 64));
    CK(cudaMalloc(&torn[i], 64));
    CK(cudaMemset(torn[i], 0, 64));
  }
  cudaStream_t s[2];
  cudaEvent_t e0[2], e1[2];
  for (int i = 0; i < 2; ++i) {
    CK(cudaSetDevice(dev[i]));
    CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[i]));
    CK(cudaEventCreate(&e1[i]));
  }
  for (int i = 0; i < 2; ++i) {
    CK(cudaSetDevice(dev[i]));
    CK(cudaEventRecord(e0[i], s[i]));
  }
  // GPU i writes into GPU 1-i's region and polls its own; done words: the
  // receiver on GPU i releases done[1-i] (the sender on GPU 1-i waits on it)
  for (int r = 1; r <= rounds; ++r)
    for (int i = 0; i < 2; ++i) {
      CK(cudaSetDevice(dev[i]));
      k_round<<<2 * C, 512, 0, s[i]>>>(reg[1 - i], reg[i], lines, (unsigned long long)r, done[1 - i], done[i], C,
                                      torn[i]);
    }
  float ms[2];
  unsigned long long h[2][2];
  for (int i = 0; i < 2; ++i) {
    CK(cudaSetDevice(dev[i]));
    CK(cudaEventRecord(e1[i], s[i]));
    CK(cudaEventSynchronize(e1[i]));
    CK(cudaEventElapsedTime(&ms[i], e0[i], e1[i]));
    CK(cudaMemcpy(h[i], torn[i], 16, cudaMemcpyDeviceToHost));
  }
  const double t = (ms[0] > ms[1] ? ms[0] : ms[1]) / 1e3;
  const double wire = (double)lines * 128 * rounds, pay = (double)lines * 120 * rounds;
  printf("LL128 probe GPU %d <-> GPU %d, %lld MiB of lines per round and direction, %d rounds, %d+%d CTAs\n", a, b,
         mib, rounds, C, C);
  printf("  per direction: wire %.1f GB/s, payload %.1f GB/s; torn 8-byte words seen: %llu / %llu\n",
         wire / t / 1e9, pay / t / 1e9, h[0][0], h[1][0]);
  return 0;
}
