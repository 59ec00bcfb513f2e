// Feasibility + bandwidth probe for NVLink SHARP multicast (NVLS) on one box,
// single process driving all visible GPUs (no handle passing needed).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
// Each GPU g multicasts a block of `bytes` (multimem.st.v4) into slot g of
// every GPU's buffer; reports per-GPU ingress GB/s and verifies the data.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CU(x)                                                                    \
  do {                                                                           \
    CUresult r = (x);                                                            \
    if (r != CUDA_SUCCESS) {                                                     \
      const char *s = nullptr;                                                   \
      cuGetErrorString(r, &s);                                                   \
      printf("FAIL %s:%d %s -> %d %s\n", __FILE__, __LINE__, #x, (int)r, s);      \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__global__ void k_fill(uint4 *p, size_t n, uint32_t tag) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = make_uint4(tag, (uint32_t)i, tag ^ 0x55u, (uint32_t)(i >> 32));
}

__global__ void k_mc_store(const uint4 *src, char *mc_dst, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint4 v = src[i];
    uint4 *d = reinterpret_cast<uint4 *>(mc_dst) + i;
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
}

// each GPU reduces its chunk across all GPUs through the switch (bf16, 8 per 16 B)
__global__ void k_mc_ld_reduce(const char *mc_src, uint4 *dst, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint4 v;
    const uint4 *s = reinterpret_cast<const uint4 *>(mc_src) + i;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(s)
                 : "memory");
    dst[i] = v;
  }
}

__global__ void k_check(const uint4 *p, size_t n, uint32_t tag, unsigned long long *bad) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint4 v = p[i];
    if (v.x != tag || v.y != (uint32_t)i || v.z != (tag ^ 0x55u)) atomicAdd(bad, 1ull);
  }
}

int main(int argc, char **argv) {
  size_t bytes = (argc > 1 ? atoll(argv[1]) : 32) << 20;  // per-GPU block
  int ctas = argc > 2 ? atoi(argv[2]) : 32;
  CU(cuInit(0));
  int ng = 0;
  cudaGetDeviceCount(&ng);
  printf("devices: %d\n", ng);
  for (int g = 0; g < ng; ++g) {
    CUdevice d;
    CU(cuDeviceGet(&d, g));
    int mc = 0, vmm = 0, fab = 0;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, d);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
    printf("dev %d: multicast=%d vmm=%d fabric=%d\n", g, mc, vmm, fab);
  }
  if (ng < 2) return 0;
  const size_t total = bytes * ng;
  std::vector<CUcontext> ctx(ng);
  for (int g = 0; g < ng; ++g) {
    CUdevice d;
    CU(cuDeviceGet(&d, g));
    CU(cuDevicePrimaryCtxRetain(&ctx[g], d));
  }
  CU(cuCtxSetCurrent(ctx[0]));
  CUmulticastObjectProp mp = {};
  mp.numDevices = ng;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = total;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t sz = (total + gran - 1) / gran * gran;
  mp.size = sz;
  printf("multicast granularity %zu, size %zu\n", gran, sz);
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int g = 0; g < ng; ++g) {
    CUdevice d;
    CU(cuDeviceGet(&d, g));
    CU(cuMulticastAddDevice(mc, d));
  }
  std::vector<CUdeviceptr> uc(ng), mcva(ng);
  for (int g = 0; g < ng; ++g) {
    CU(cuCtxSetCurrent(ctx[g]));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ag = 0;
    CU(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle mem;
    CU(cuMemCreate(&mem, sz, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, mem, 0, sz, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = g;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemAddressReserve(&uc[g], sz, ag, 0, 0));
    CU(cuMemMap(uc[g], sz, 0, mem, 0));
    CU(cuMemSetAccess(uc[g], sz, &acc, 1));
    CU(cuMemAddressReserve(&mcva[g], sz, gran, 0, 0));
    CU(cuMemMap(mcva[g], sz, 0, mc, 0));
    CU(cuMemSetAccess(mcva[g], sz, &acc, 1));
  }
  printf("bound + mapped on %d GPUs\n", ng);
  std::vector<uint4 *> src(ng);
  std::vector<cudaStream_t> st(ng);
  for (int g = 0; g < ng; ++g) {
    cudaSetDevice(g);
    cudaMalloc(&src[g], bytes);
    cudaStreamCreate(&st[g]);
    k_fill<<<1024, 256, 0, st[g]>>>(src[g], bytes / 16, 1000 + g);
  }
  for (int g = 0; g < ng; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); }
  // timed: every GPU multicasts its block concurrently
  for (int rep = 0; rep < 3; ++rep) {
    std::vector<cudaEvent_t> e0(ng), e1(ng);
    for (int g = 0; g < ng; ++g) {
      cudaSetDevice(g);
      cudaEventCreate(&e0[g]);
      cudaEventCreate(&e1[g]);
      cudaEventRecord(e0[g], st[g]);
      for (int it = 0; it < 10; ++it)
        k_mc_store<<<ctas, 512, 0, st[g]>>>(src[g], (char *)mcva[g] + (size_t)g * bytes, bytes / 16);
      cudaEventRecord(e1[g], st[g]);
    }
    double worst = 0;
    for (int g = 0; g < ng; ++g) {
      cudaSetDevice(g);
      cudaEventSynchronize(e1[g]);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0[g], e1[g]);
      worst = ms / 10 > worst ? ms / 10 : worst;
    }
    printf("rep %d: %zu MiB/GPU multicast to %d GPUs in %.1f us -> ingress %.1f GB/s per GPU (ctas %d)\n", rep,
           bytes >> 20, ng, worst * 1e3, (double)bytes * (ng - 1) / (worst * 1e-3) / 1e9, ctas);
  }
  // reduce-scatter through the switch: GPU g reads chunk g (bytes) of the
  // multicast buffer with ld_reduce; busbw = (ng-1)/ng * (ng*bytes) / t
  for (int rep = 0; rep < 3; ++rep) {
    std::vector<cudaEvent_t> e0(ng), e1(ng);
    for (int g = 0; g < ng; ++g) {
      cudaSetDevice(g);
      cudaEventCreate(&e0[g]);
      cudaEventCreate(&e1[g]);
      cudaEventRecord(e0[g], st[g]);
      for (int it = 0; it < 10; ++it)
        k_mc_ld_reduce<<<ctas, 512, 0, st[g]>>>((const char *)mcva[g] + (size_t)g * bytes, src[g], bytes / 16);
      cudaEventRecord(e1[g], st[g]);
    }
    double worst = 0;
    for (int g = 0; g < ng; ++g) {
      cudaSetDevice(g);
      cudaEventSynchronize(e1[g]);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0[g], e1[g]);
      worst = ms / 10 > worst ? ms / 10 : worst;
    }
    printf("rep %d: ld_reduce bf16 chunk %zu MiB/GPU from %d GPUs in %.1f us -> RS busbw %.1f GB/s (ctas %d)\n", rep,
           bytes >> 20, ng, worst * 1e3, (double)bytes * (ng - 1) / (worst * 1e-3) / 1e9, ctas);
  }
  for (int g = 0; g < ng; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); }
  unsigned long long *bad;
  cudaMallocManaged(&bad, 8);
  *bad = 0;
  for (int g = 0; g < ng; ++g) {
    cudaSetDevice(g);
    for (int q = 0; q < ng; ++q)
      k_check<<<1024, 256>>>(reinterpret_cast<uint4 *>(uc[g] + (size_t)q * bytes), bytes / 16, 1000 + q, bad);
    cudaDeviceSynchronize();
  }
  printf("verify: %llu bad vectors\n", *bad);
  return 0;
}
