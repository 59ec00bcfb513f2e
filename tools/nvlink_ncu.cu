// NVLink evidence for the collectives' data paths under ncu (one process).
//
// A collective kernel waits on its peers, so ncu cannot replay it (replays
// serialise the GPUs and the peers never arrive). This binary runs the SAME
// device loops the collectives use — store_units (push: AG direct/ring/rec
// push), copy_units (pull: AG pull kernels), reduce2_units (pull + fused add:
// RS ring/recursive pull step) — from GPU 0 against peer memory of GPUs
// 1..n-1 mapped with cudaDeviceEnablePeerAccess, with no flags, so ncu can
// replay them and read nvltx/nvlrx byte counters.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/nvlink_ncu tools/nvlink_ncu.cu
//   tools/nvlink_ncu                       # device-timed GB/s per pattern
//   ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,... tools/nvlink_ncu --once
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2504_18658_b200/csrc/kernels.cuh"

using namespace pccl;

#define CHECK(x)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) {                                                                  \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));      \
      exit(1);                                                                                \
    }                                                                                         \
  } while (0)

struct Peers {
  char *p[PCCL_MAXR];
  int n;
};

// AG direct push data path: my block -> every peer's recv (store_units).
__global__ void __launch_bounds__(kThreads) k_push(const char *src, Peers dst, int64_t units) {
  int64_t lo, hi;
  split32(units, gridDim.x, blockIdx.x, lo, hi);
  for (int i = 0; i < dst.n; ++i) store_units<16>(dst.p[(blockIdx.x + i) % dst.n], src, lo, hi);
}
// AG pull data path: every peer's block -> my recv (copy_units, LDG .cg).
__global__ void __launch_bounds__(kThreads) k_pull(char *dst, Peers src, int64_t units) {
  int64_t lo, hi;
  split32(units, gridDim.x, blockIdx.x, lo, hi);
  for (int i = 0; i < src.n; ++i)
    copy_units<16, kUnroll>(dst + (int64_t)i * units * 16, src.p[(blockIdx.x + i) % src.n], lo, hi);
}
// RS recursive-halving pull step: work = own + partner (bf16, fp32 accumulate).
__global__ void __launch_bounds__(kThreads) k_pull_reduce(char *dst, const char *own, Peers src, int64_t units) {
  int64_t lo, hi;
  split32(units, gridDim.x, blockIdx.x, lo, hi);
  reduce2_units<DT_BF16, true, kUnroll>(dst, own, src.p[0], lo, hi);
}

int main(int argc, char **argv) {
  const bool once = argc > 1 && !strcmp(argv[1], "--once");
  int ngpu = 0;
  CHECK(cudaGetDeviceCount(&ngpu));
  if (ngpu < 2) {
    fprintf(stderr, "needs >= 2 GPUs\n");
    return 1;
  }
  const size_t B = (size_t)64 << 20;  // bytes per peer
  const int64_t units = (int64_t)(B / 16);
  Peers peers = {};
  peers.n = ngpu - 1;
  CHECK(cudaSetDevice(0));
  for (int g = 1; g < ngpu; ++g) {
    CHECK(cudaDeviceEnablePeerAccess(g, 0));
    CHECK(cudaSetDevice(g));
    CHECK(cudaMalloc(&peers.p[g - 1], B));
    CHECK(cudaMemset(peers.p[g - 1], g, B));
    CHECK(cudaSetDevice(0));
  }
  char *local = nullptr, *out = nullptr;
  CHECK(cudaMalloc(&local, B));
  CHECK(cudaMalloc(&out, B * (size_t)peers.n));
  CHECK(cudaMemset(local, 1, B));
  CHECK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CHECK(cudaEventCreate(&a));
  CHECK(cudaEventCreate(&b));
  Peers one = peers;
  one.n = 1;
  struct Case {
    const char *name;
    int which;
    double bytes;  // algorithmic NVLink bytes per launch (one direction)
  } cases[] = {{"push_all_peers (AG direct push)", 0, (double)B * peers.n},
               {"pull_all_peers (AG direct pull)", 1, (double)B * peers.n},
               {"pull_reduce_one_peer (RS rechalf step, bf16)", 2, (double)B}};
  const int ctas = 128;
  for (const Case &cs : cases) {
    auto launch = [&]() {
      if (cs.which == 0) k_push<<<ctas, kThreads>>>(local, peers, units);
      else if (cs.which == 1) k_pull<<<ctas, kThreads>>>(out, peers, units);
      else k_pull_reduce<<<ctas, kThreads>>>(out, local, one, units);
    };
    const int iters = once ? 1 : 20;
    launch();
    CHECK(cudaDeviceSynchronize());
    CHECK(cudaEventRecord(a));
    for (int i = 0; i < iters; ++i) launch();
    CHECK(cudaEventRecord(b));
    CHECK(cudaEventSynchronize(b));
    float ms = 0;
    CHECK(cudaEventElapsedTime(&ms, a, b));
    const double t = ms * 1e-3 / iters;
    printf("%-46s %d peer(s) %8.1f us  %7.1f GB/s algorithmic NVLink\n", cs.name, cs.which == 2 ? 1 : peers.n,
           t * 1e6, cs.bytes / t / 1e9);
  }
  CHECK(cudaGetLastError());
  return 0;
}
