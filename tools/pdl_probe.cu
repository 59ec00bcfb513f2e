// Kernel-boundary cost under programmatic dependent launch, per GPU, no
// communication: K back-to-back launches of a kernel that only passes
// griddepcontrol.wait / launch_dependents, with optional system-scope memory
// operations in its body, timed with events. Tells whether the 1-5 us
// "completion -> dependent release" seen between the collectives
// (tools/trace_seq.py: epi->pdl) is a property of the GPU or of what the
// kernel does.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/pdl_probe tools/pdl_probe.cu
//   tools/pdl_probe [device ...]
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

// mode 0: nothing; 1: thread 0 of every CTA st.release.sys to local memory;
// 2: fence.sc.sys; 3: st.relaxed.sys to PEER memory (if peer != null);
// 4: st.release.sys to peer memory; 5: 1 MiB of local stores per CTA
__global__ void k_body(unsigned long long *local, unsigned long long *peer, int mode, char *buf) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (mode == 5) {
    uint4 *b = reinterpret_cast<uint4 *>(buf) + (size_t)blockIdx.x * (1 << 16);
    for (int i = threadIdx.x; i < (1 << 16); i += blockDim.x) b[i] = make_uint4(i, i, i, i);
  }
  if (mode >= 8 && mode <= 11 && peer) {  // 64 KiB of data stores into the peer per CTA
    uint4 *b = reinterpret_cast<uint4 *>(peer + 4096) + (size_t)blockIdx.x * 4096;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) b[i] = make_uint4(i, i, i, i);
  }
  if (mode == 13 && peer) {  // 64 KiB of data loads from the peer per CTA
    const uint4 *b = reinterpret_cast<const uint4 *>(peer + 4096) + (size_t)blockIdx.x * 4096;
    uint32_t acc = 0;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) acc ^= __ldcg(b + i).x;
    if (acc == 0x12345678u) local[2048] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long *w = local + blockIdx.x;
    if (mode == 12 && peer) {
      unsigned long long v;
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(peer + blockIdx.x) : "memory");
      if (v == 0x1234567ull) local[2049] = v;
    }
    if (mode == 6) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (mode == 7) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(w), "l"(1ull) : "memory");
    if (mode == 8 && peer) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer + blockIdx.x), "l"(1ull) : "memory");
    if (mode == 9 && peer) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(peer + blockIdx.x), "l"(1ull) : "memory");
    }
    if (mode == 11 && peer) {  // gpu-scope release into a local counter; the last CTA publishes with release.sys
      unsigned long long old;
      asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(local + 1024) : "memory");
      if ((old + 1) % gridDim.x == 0)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer + 2048), "l"(old) : "memory");
    }
    if (mode == 1) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(w), "l"(1ull) : "memory");
    if (mode == 2) asm volatile("fence.sc.sys;" ::: "memory");
    if (mode == 3 && peer) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(peer + blockIdx.x), "l"(1ull) : "memory");
    if (mode == 4 && peer) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer + blockIdx.x), "l"(1ull) : "memory");
  }
}

static int g_domain = 0;  // 1: launch in the "remote" memory-synchronization domain
static float run_eager(int mode, int ctas, int threads, bool pdl, unsigned long long *local,
                       unsigned long long *peer, char *buf, cudaStream_t s) {
  const int K = 1000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeMemSyncDomain;
  attr[1].val.memSyncDomain = g_domain ? cudaLaunchMemSyncDomainRemote : cudaLaunchMemSyncDomainDefault;
  if (!pdl) attr[0] = attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = (pdl ? 1 : 0) + 1;
  // a long first kernel lets the host queue all K launches before they run
  for (int i = 0; i < 20; ++i) CK(cudaLaunchKernelEx(&cfg, k_body, local, peer, mode, buf));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaStreamSynchronize(s));
  cudaLaunchConfig_t big = cfg;
  big.gridDim = dim3(148);
  big.numAttrs = 0;
  for (int i = 0; i < 40; ++i) CK(cudaLaunchKernelEx(&big, k_body, local, peer, 5, buf));  // ~1 ms of local stores
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < K; ++i) CK(cudaLaunchKernelEx(&cfg, k_body, local, peer, mode, buf));
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms * 1e3f / K;
}

// K launches of a ONE-kernel graph (what an eager API could do per call)
static float run_graph1(int mode, int ctas, int threads, bool pdl, unsigned long long *local,
                        unsigned long long *peer, char *buf, cudaStream_t s) {
  const int K = 1000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  CK(cudaLaunchKernelEx(&cfg, k_body, local, peer, mode, buf));
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int i = 0; i < 20; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  cudaLaunchConfig_t big = cfg;
  big.gridDim = dim3(148);
  big.numAttrs = 0;
  for (int i = 0; i < 40; ++i) CK(cudaLaunchKernelEx(&big, k_body, local, peer, 5, buf));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < K; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(g));
  return ms * 1e3f / K;
}

static float run(int mode, int ctas, int threads, bool pdl, unsigned long long *local, unsigned long long *peer,
                 char *buf, cudaStream_t s) {
  const int K = 1000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  for (int i = 0; i < 20; ++i) CK(cudaLaunchKernelEx(&cfg, k_body, local, peer, mode, buf));
  // capture K launches in a graph so host launch cost is out of the picture
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < K; ++i) CK(cudaLaunchKernelEx(&cfg, k_body, local, peer, mode, buf));
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, s));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(g));
  return ms * 1e3f / K;
}

int main(int argc, char **argv) {
  int n;
  CK(cudaGetDeviceCount(&n));
  const char *names[] = {"empty", "st.release.sys local", "fence.sc.sys", "st.relaxed.sys peer",
                         "st.release.sys peer", "1 MiB local stores", "fence.acq_rel.gpu", "st.release.gpu local",
                         "64K peer st + rel.sys", "64K peer st + gpu fence", "64K peer st only",
                         "64K peer st + 1 rel.sys", "ld.relaxed.sys peer", "64K peer ld.cg"};
  for (int ai = 1; ai <= (argc > 1 ? argc - 1 : n); ++ai) {
    const int d = argc > 1 ? atoi(argv[ai]) : ai - 1;
    const int peer_dev = n > 1 ? (d + 1) % n : -1;
    CK(cudaSetDevice(d));
    unsigned long long *local, *peer = nullptr;
    char *buf;
    CK(cudaMalloc(&local, 4096 * 8));
    CK(cudaMalloc(&buf, (size_t)148 << 20));
    if (peer_dev >= 0) {
      int ok = 0;
      CK(cudaDeviceCanAccessPeer(&ok, d, peer_dev));
      if (ok) {
        cudaError_t e = cudaDeviceEnablePeerAccess(peer_dev, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
        CK(cudaSetDevice(peer_dev));
        CK(cudaMalloc(&peer, (size_t)(4096 * 8) + ((size_t)128 << 16)));
        CK(cudaSetDevice(d));
      }
    }
    // the same peer memory again, but allocated and mapped through the VMM API
    // (cuMemCreate on the peer + cuMemMap, access granted to this device)
    unsigned long long *vpeer = nullptr;
    if (peer) {
      CUmemAllocationProp prop = {};
      prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      prop.location.id = peer_dev;
      size_t gran = 0;
      cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
      const size_t bytes = ((((size_t)(4096 * 8) + ((size_t)128 << 16)) + gran - 1) / gran) * gran;
      CUmemGenericAllocationHandle h;
      CUdeviceptr va;
      if (cuMemCreate(&h, bytes, &prop, 0) == CUDA_SUCCESS && cuMemAddressReserve(&va, bytes, gran, 0, 0) == CUDA_SUCCESS &&
          cuMemMap(va, bytes, 0, h, 0) == CUDA_SUCCESS) {
        CUmemAccessDesc acc[2] = {};
        acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[0].location.id = d;
        acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        acc[1] = acc[0];
        acc[1].location.id = peer_dev;
        if (cuMemSetAccess(va, bytes, acc, 2) == CUDA_SUCCESS) vpeer = (unsigned long long *)va;
      }
      if (!vpeer) printf("  (VMM peer mapping failed)\n");
    }
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaDeviceProp pr;
    CK(cudaGetDeviceProperties(&pr, d));
    printf("GPU %d (bus %02x, peer GPU %d): us per launch in a graph of 1000\n", d, pr.pciBusID, peer_dev);
    for (int mode = 0; mode < 14; ++mode) {
      if (mode == 5 || mode == 1 || mode == 2 || mode == 6 || mode == 7) continue;
      const float a = run(mode, 1, 32, true, local, peer, buf, s);
      const float b = run(mode, 128, 512, true, local, peer, buf, s);
      const float c = run(mode, 128, 512, false, local, peer, buf, s);
      const float e = run_eager(mode, 128, 512, true, local, peer, buf, s);
      const float f = vpeer ? run_eager(mode, 128, 512, true, local, vpeer, buf, s) : -1.f;
      const float gv = vpeer ? run(mode, 128, 512, true, local, vpeer, buf, s) : -1.f;
      g_domain = 1;
      const float h = run_eager(mode, 128, 512, true, local, peer, buf, s);
      g_domain = 0;
      printf("  %-22s  1x32 pdl %6.2f   128x512 pdl %6.2f   no-pdl %6.2f   eager pdl %6.2f   eager remote-domain %6.2f"
             "   VMM peer: graph %6.2f eager %6.2f\n", names[mode], a, b, c, e, h, gv, f);
    }
    CK(cudaStreamDestroy(s));
  }
  return 0;
}
