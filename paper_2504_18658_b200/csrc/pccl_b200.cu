// pccl_b200.cu — C-ABI implementation: worlds (symmetric segments over CUDA
// IPC), communicators (flag slots + epochs), call planning (staging, layout,
// vector width, grid) and kernel dispatch. See include/pccl_b200.h.
#include "../../include/pccl_b200.h"
#include "kernels.cuh"

#include <cuda.h>  // driver types for the stream memory operations (entry points via cudart)

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <mutex>
#include <deque>
#include <thread>
#include <chrono>
#include <type_traits>
#include <vector>

using namespace pccl;

namespace {

constexpr int kMaxSegs = 1024;

struct Segment {
  bool used = false;
  size_t bytes = 0;
  char *ptr[PCCL_MAXR] = {};      // valid in this process (own, peer-mapped or emulated)
  bool opened[PCCL_MAXR] = {};    // cudaIpcOpenMemHandle'd (must be closed)
  bool owned[PCCL_MAXR] = {};     // cudaMalloc'd here (must be freed)
  bool reg = false;               // caller-owned memory registered collectively (pccl_segment_register)
  char *ipc_base[PCCL_MAXR] = {}; // registered: peer allocation base opened through the world's IPC cache
};

}  // namespace

struct OccKey {
  const void *k;
  int threads;
  size_t smem;
  bool operator<(const OccKey &o) const {
    return k != o.k ? k < o.k : threads != o.threads ? threads < o.threads : smem < o.smem;
  }
};

// Point-to-point state of one world rank executed by this process.
struct P2PMsg {
  int64_t tag = 0;
  size_t bytes = 0;
  char *dev = nullptr;  // cudaMalloc'd copy (complete message), nullptr when bytes == 0
  size_t have = 0;      // fragment assembly: bytes received so far
};
struct P2PRank {
  uint64_t head_sent[PCCL_MAXR] = {};  // bytes I wrote into rank q's ring from me
  uint64_t tail_read[PCCL_MAXR] = {};  // bytes I consumed from my ring of source q
  std::deque<P2PMsg> unexpected[PCCL_MAXR];  // complete messages from source q, arrival order
  P2PMsg partial[PCCL_MAXR];                 // message from q being assembled (fragments)
  bool in_partial[PCCL_MAXR] = {};
  cudaStream_t stream = nullptr;
  char *hdr = nullptr;  // pinned 64-byte scratch
};

struct pccl_world {
  int nranks = 0;
  int rank = -1;  // -1: emulation
  int device = 0;
  bool emu = false;
  Segment segs[kMaxSegs];
  int seg_hi = 1;  // one past the highest segment index ever used (bounds the resolve() scan)
  int staging = -1;
  volatile int *err_host = nullptr;
  int *err_dev = nullptr;
  uint64_t epoch[PCCL_NSLOTS] = {};
  uint64_t ce_calls[PCCL_NSLOTS] = {};  // copy-engine collectives per group (host-issued, never captured)
  struct NvlsSeg {  // multicast segment (NVLS): this rank's physical memory bound to a switch multicast object
    bool used = false, bound = false;
    unsigned long long mc = 0, mem = 0;  // CUmemGenericAllocationHandle
    unsigned long long mc_va = 0, uc_va = 0;
    size_t bytes = 0, gran = 0;  // gran: multicast granularity (VA alignment of both mappings)
  } nvls[4];
  std::map<uint32_t, int> slot_of_mask;  // emulation: dynamic slot allocation
  int sms = 148;
  // tuning knobs (pccl_world_set_param)
  int64_t p_ctas = 0;  // 0: auto
  int64_t p_nsub = 1;
  int64_t p_threads = 512;
  int64_t p_ag_variant = -1;  // -1: auto (per algorithm / buffer registration)
  int64_t p_rs_variant = -1;
  int64_t p_tma_stages = 3;
  int64_t p_tma_tile = 65536;
  int64_t p_timeout_ms = 20000;
  int64_t p_trace = 0;
  int poisoned = 0;  // sticky device error
  int64_t p_pdl = 1;          // programmatic dependent launch between back-to-back collectives
  int64_t p_local_fence = 1;  // pull-kernel signals: gpu-scope fence + relaxed sys store (see device.cuh)
  int64_t p_item_kib = 0;
  int64_t p_items_per_cta = 2;  // rs_variant 7: work items per CTA per step
  int64_t p_hier_intra = -1;    // hierarchical intra phase: -1 auto (direct for M >= 3), 0 ring, 1 direct
  int64_t p_hier_chain = 1;     // hierarchical: chain the two phase launches (device.cuh "chained launches")  // direct kernels: dynamically claimed work items of this size (0: static CTA slices)
  int64_t p_staged_bytes = 0;  // statistic: bytes of caller buffers bound through staging (get_param; set 0 = reset)
  int64_t p_ll_max = -1;  // LL protocol up to this many payload bytes per peer; 0 off, -1 auto (kLLEgress / (gs-1))
  // LL128 (direct AG) up to this many payload bytes per peer where LL does not
  // apply; 0 off. Default: whatever one region holds (tools/tune.py, p=2/4,
  // 1-7 MiB: never slower than the flag protocol, up to 1.7x at p=2 / 3 MiB)
  int64_t p_ll128_max = (int64_t)PCCL_LL128_MAX_PAYLOAD;
  uint64_t *trace_buf = nullptr;  // device, PCCL_MAXR x PCCL_MAX_CTAS x PCCL_TRACE_EVENTS
  int trace_rows = 0, trace_ctas = 0;
  int64_t trace_seq = 0;  // launches traced since tracing was (re)enabled
  uint32_t meta_skew[PCCL_MAXR] = {};
  std::map<uint32_t, pccl_comm *> comm_cache;  // hierarchical sub-groups
  std::map<OccKey, int> occ_cache;              // co-resident CTAs per SM, per (kernel, threads, smem)
  std::map<std::string, std::pair<char *, int>> ipc_open;  // (peer, allocation handle) -> (mapped base, refs)
  P2PRank p2p[PCCL_MAXR];  // indexed by world rank (real mode: own rank only)
  std::mutex occ_mu;
};

struct pccl_comm {
  pccl_world *w = nullptr;
  int gs = 0;
  int members[PCCL_MAXR] = {};
  int gi = -1;  // this process's index (real mode)
  int slot = 0;
  int comm_id = 0;
  uint32_t mask = 0;
};

namespace {

int cuda_err(cudaError_t e) {
  if (e == cudaSuccess) return PCCL_SUCCESS;
  fprintf(stderr, "[pccl_b200] CUDA error: %s\n", cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? PCCL_ERR_OUT_OF_MEMORY : PCCL_ERR_CUDA;
}
#define CK(x)                                 \
  do {                                        \
    int _s = cuda_err(x);                     \
    if (_s != PCCL_SUCCESS) return _s;        \
  } while (0)

size_t dt_size(int dt) {
  switch (dt) {
    case PCCL_FLOAT32: return 4;
    case PCCL_BFLOAT16: return 2;
    case PCCL_FLOAT16: return 2;
    case PCCL_UINT8: return 1;
    case PCCL_INT32: return 4;
    case PCCL_INT64: return 8;
    case PCCL_FLOAT64: return 8;
  }
  return 0;
}
bool is_pow2(int x) { return x >= 1 && (x & (x - 1)) == 0; }
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

uint32_t hash_meta(int coll, int algo, int order, size_t count, int dtype, int gs) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h ^= v; h *= 1099511628211ull; };
  mix(coll); mix(algo); mix(order); mix(count); mix(dtype); mix(gs);
  return (uint32_t)(h ^ (h >> 32)) & 0x7fffffff;
}

int slot_for(pccl_world *w, uint32_t mask) {
  if (!w->emu) return (int)mask;  // real mode: nranks <= 8 -> mask < 256
  auto it = w->slot_of_mask.find(mask);
  if (it != w->slot_of_mask.end()) return it->second;
  int s = (int)w->slot_of_mask.size();
  if (s >= PCCL_NSLOTS) return -1;
  w->slot_of_mask[mask] = s;
  return s;
}

// Find (segment, offset) of a pointer owned by world rank r.
bool resolve(pccl_world *w, int r, const void *p, size_t bytes, int *seg, size_t *off) {
  const char *c = (const char *)p;
  for (int s = 1; s < w->seg_hi; ++s) {
    const Segment &S = w->segs[s];
    if (!S.used || !S.ptr[r]) continue;
    if (c >= S.ptr[r] && c + bytes <= S.ptr[r] + S.bytes) {
      *seg = s;
      *off = (size_t)(c - S.ptr[r]);
      return true;
    }
  }
  return false;
}

int max_coresident(const void *kernel, int threads, int sms) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess) return sms;
  return std::max(1, per_sm) * sms;
}

// --------------------------------------------------------------------------
// kernel selection
// --------------------------------------------------------------------------
using KernelFn = void (*)(LaunchParams);

KernelFn ag_kernel(int algo, int U) {
#define AGK(A, K)                              \
  if (algo == A) {                             \
    switch (U) {                               \
      case 16: return (KernelFn)K<16>;         \
      case 8: return (KernelFn)K<8>;           \
      case 4: return (KernelFn)K<4>;           \
      case 2: return (KernelFn)K<2>;           \
      default: return (KernelFn)K<1>;          \
    }                                          \
  }
  AGK(A_DIRECT, k_ag_direct)
  AGK(A_RING, k_ag_ring)
  AGK(A_REC, k_ag_rec)
#undef AGK
  return nullptr;
}

template <int DT, bool VEC>
KernelFn rs_direct_pp_kernel(int order, int maxp) {
#define RSP(O)                                                          \
  if (order == O) {                                                     \
    if (!VEC) return (KernelFn)k_rs_direct_pp<DT, VEC, O, 16>;          \
    switch (maxp) {                                                     \
      case 2: return (KernelFn)k_rs_direct_pp<DT, VEC, O, 2>;           \
      case 4: return (KernelFn)k_rs_direct_pp<DT, VEC, O, 4>;           \
      case 8: return (KernelFn)k_rs_direct_pp<DT, VEC, O, 8>;           \
      default: return (KernelFn)k_rs_direct_pp<DT, VEC, O, 16>;         \
    }                                                                   \
  }
  RSP(O_RING)
  RSP(O_REC)
  RSP(O_RANK)
#undef RSP
  return nullptr;
}

template <int DT, bool VEC, bool PUSH>
KernelFn rs_direct_kernel(int order, int maxp) {
#define RSD(O)                                                          \
  if (order == O) {                                                     \
    if (!VEC) return (KernelFn)k_rs_direct<DT, VEC, O, 16, PUSH>;       \
    switch (maxp) {                                                     \
      case 2: return (KernelFn)k_rs_direct<DT, VEC, O, 2, PUSH>;        \
      case 4: return (KernelFn)k_rs_direct<DT, VEC, O, 4, PUSH>;        \
      case 8: return (KernelFn)k_rs_direct<DT, VEC, O, 8, PUSH>;        \
      default: return (KernelFn)k_rs_direct<DT, VEC, O, 16, PUSH>;      \
    }                                                                   \
  }
  RSD(O_RING)
  RSD(O_REC)
  RSD(O_RANK)
#undef RSD
  return nullptr;
}

template <int DT, bool VEC>
KernelFn rs_kernel_dt(int algo, int order, int maxp, int variant) {
  if (algo == A_RING) return variant == 1 ? (KernelFn)k_rs_ring_push<DT, VEC> : (KernelFn)k_rs_ring<DT, VEC>;
  if (algo == A_REC)
    return variant == 1 ? (KernelFn)k_rs_rec_push<DT, VEC>
                        : variant == 7 ? (KernelFn)k_rs_rec_items<DT, VEC> : (KernelFn)k_rs_rec<DT, VEC>;
  if (variant == 5) return rs_direct_pp_kernel<DT, VEC>(order, maxp);
  return variant == 1 ? rs_direct_kernel<DT, VEC, true>(order, maxp) : rs_direct_kernel<DT, VEC, false>(order, maxp);
}

template <int DT>
KernelFn rs_ll_dt(int order, int maxp) {
#define RLL(O)                                                  \
  if (order == O) {                                             \
    switch (maxp) {                                             \
      case 2: return (KernelFn)k_rs_direct_ll<DT, O, 2>;        \
      case 4: return (KernelFn)k_rs_direct_ll<DT, O, 4>;        \
      case 8: return (KernelFn)k_rs_direct_ll<DT, O, 8>;        \
      default: return (KernelFn)k_rs_direct_ll<DT, O, 16>;      \
    }                                                           \
  }
  RLL(O_RING)
  RLL(O_REC)
  RLL(O_RANK)
#undef RLL
  return nullptr;
}
template <int DT>
KernelFn rs_ll128_dt(int order, int maxp) {
#define RLL(O)                                                    \
  if (order == O) {                                               \
    switch (maxp) {                                               \
      case 2: return (KernelFn)k_rs_direct_ll128<DT, O, 2>;       \
      case 4: return (KernelFn)k_rs_direct_ll128<DT, O, 4>;       \
      case 8: return (KernelFn)k_rs_direct_ll128<DT, O, 8>;       \
      default: return (KernelFn)k_rs_direct_ll128<DT, O, 16>;     \
    }                                                             \
  }
  RLL(O_RING)
  RLL(O_REC)
  RLL(O_RANK)
#undef RLL
  return nullptr;
}
KernelFn rs_ll128_kernel(int dt, int order, int maxp) {
  if (dt == PCCL_FLOAT32) return rs_ll128_dt<DT_F32>(order, maxp);
  if (dt == PCCL_BFLOAT16) return rs_ll128_dt<DT_BF16>(order, maxp);
  if (dt == PCCL_FLOAT16) return rs_ll128_dt<DT_F16>(order, maxp);
  return nullptr;
}
KernelFn rs_ll_kernel(int dt, int order, int maxp) {
  if (dt == PCCL_FLOAT32) return rs_ll_dt<DT_F32>(order, maxp);
  if (dt == PCCL_BFLOAT16) return rs_ll_dt<DT_BF16>(order, maxp);
  if (dt == PCCL_FLOAT16) return rs_ll_dt<DT_F16>(order, maxp);
  return nullptr;
}

KernelFn rs_kernel(int dt, bool vec, int algo, int order, int maxp, int variant) {
#define RSK(D)                                                                                              \
  return vec ? rs_kernel_dt<D, true>(algo, order, maxp, variant) : rs_kernel_dt<D, false>(algo, order, maxp, variant);
  if (dt == PCCL_FLOAT32) { RSK(DT_F32) }
  if (dt == PCCL_BFLOAT16) { RSK(DT_BF16) }
  if (dt == PCCL_FLOAT16) { RSK(DT_F16) }
#undef RSK
  return nullptr;
}

// --------------------------------------------------------------------------
// a planned launch: rows (world ranks acted for) and their groups
// --------------------------------------------------------------------------
struct Row {
  int rank;              // world rank
  const pccl_comm *g;    // its group
};

struct Plan {
  int coll;  // 0 AG, 1 RS
  int algo;
  int order = 0;
  int dtype;
  size_t count;          // AG: elements per member block; RS: elements per chunk
  int gs;
  std::vector<Row> rows;
  // layout in ELEMENTS (converted to units at launch)
  int nsubblk = 1;
  int64_t blk = 0, sub_stride = 0, istride = 0, send_sub_stride = 0, out_sub_stride = 0;
  int64_t base[PCCL_MAXR] = {};  // by world rank
  int local_copy = 1;
  // per world rank buffers
  char *send[PCCL_MAXR] = {}, *recv[PCCL_MAXR] = {}, *work[PCCL_MAXR] = {}, *out[PCCL_MAXR] = {};
  uint32_t place = 0;  // symmetric-placement hash (real mode)
  int variant = 0;
  int wire = 0;        // direct RS: round after every add (step-wise rounding points)
  int rank_final = 0;  // push AG final unit published rank-level (flat calls)
  int chain = 0;       // chained pair (device.cuh): 1 first launch, 2 second launch
  uint32_t chain_slot_off[PCCL_MAXR] = {};  // chain 1, per row: the second group's slot (words)
  int force_ctas = 0;  // > 0: CTAs per row (chained launches must cut identical slices)
};

int launch(pccl_world *w, Plan &pl, cudaStream_t stream) {
  const size_t es = dt_size(pl.dtype);
  LaunchParams P;
  memset(&P, 0, sizeof(P));
  P.gs = pl.gs;
  P.nsubblk = pl.nsubblk;
  P.local_copy = pl.local_copy;
  P.order = pl.order;
  P.timeout_ns = (w->p_timeout_ms * 1000000ll);
  P.err = w->err_dev;
  P.nsub = (int)std::max<int64_t>(1, std::min<int64_t>(w->p_nsub, 32));
  P.variant = pl.variant;
  P.local_fence = (int)w->p_local_fence;
  P.wire = pl.wire;
  P.chain = pl.chain;
  P.rank_final = pl.rank_final;
  P.tma_stages = (int)w->p_tma_stages;
  P.tma_tile = (uint32_t)w->p_tma_tile;

  // ---- unit size: largest power of two dividing every byte offset/pointer
  const int64_t bytes_terms[] = {pl.blk * (int64_t)es, pl.sub_stride * (int64_t)es, pl.istride * (int64_t)es,
                                 pl.send_sub_stride * (int64_t)es, pl.out_sub_stride * (int64_t)es};
  uint64_t acc = 0;
  for (int64_t t : bytes_terms) acc |= (uint64_t)t;
  for (const Row &rw : pl.rows) {
    acc |= (uint64_t)(pl.base[rw.rank] * (int64_t)es);
    for (int m = 0; m < rw.g->gs; ++m) {
      const int q = rw.g->members[m];
      for (char *p : {pl.send[q], pl.recv[q], pl.work[q], pl.out[q]}) acc |= (uint64_t)(uintptr_t)p;
    }
  }
  int U;  // bytes per unit
  KernelFn k;
  size_t smem = 0;
  if (pl.variant == 8) {  // LL128 line protocol (direct collectives), 8-byte payload units
    U = 8;
    int maxp = 2;
    while (maxp < pl.gs) maxp <<= 1;
    if (pl.coll == PCCL_ALL_GATHER) {
      switch (maxp) {
        case 2: k = (KernelFn)k_ag_direct_ll128<2>; break;
        case 4: k = (KernelFn)k_ag_direct_ll128<4>; break;
        case 8: k = (KernelFn)k_ag_direct_ll128<8>; break;
        default: k = (KernelFn)k_ag_direct_ll128<16>; break;
      }
    } else {
      k = rs_ll128_kernel(pl.dtype, pl.order, maxp);
    }
  } else if (pl.variant == 4) {  // LL protocol: 8-byte payload units (host checked the alignment)
    U = 8;
    int maxp = 2;
    while (maxp < pl.gs) maxp <<= 1;
    if (pl.coll == PCCL_ALL_GATHER) {
      switch (maxp) {
        case 2: k = (KernelFn)k_ag_direct_ll<2>; break;
        case 4: k = (KernelFn)k_ag_direct_ll<4>; break;
        case 8: k = (KernelFn)k_ag_direct_ll<8>; break;
        default: k = (KernelFn)k_ag_direct_ll<16>; break;
      }
    } else {
      k = rs_ll_kernel(pl.dtype, pl.order, maxp);
    }
  } else if (pl.coll == PCCL_ALL_GATHER) {
    U = 16;
    while (U > 1 && (acc & (uint64_t)(U - 1))) U >>= 1;
    if ((size_t)U < es && es <= 16 && !(acc & (es - 1))) U = (int)es;
    k = ag_kernel(pl.algo, U);
    if (pl.variant == 1 && pl.algo == A_RING) {
      switch (U) {
        case 16: k = (KernelFn)k_ag_ring_push<16>; break;
        case 8: k = (KernelFn)k_ag_ring_push<8>; break;
        case 4: k = (KernelFn)k_ag_ring_push<4>; break;
        case 2: k = (KernelFn)k_ag_ring_push<2>; break;
        default: k = (KernelFn)k_ag_ring_push<1>; break;
      }
    }
    if (pl.variant == 1 && pl.algo == A_REC) {
      switch (U) {
        case 16: k = (KernelFn)k_ag_rec_push<16>; break;
        case 8: k = (KernelFn)k_ag_rec_push<8>; break;
        case 4: k = (KernelFn)k_ag_rec_push<4>; break;
        case 2: k = (KernelFn)k_ag_rec_push<2>; break;
        default: k = (KernelFn)k_ag_rec_push<1>; break;
      }
    }
    if (pl.algo == A_DIRECT && (pl.variant == 1 || pl.variant == 3))
      k = U == 16 ? (KernelFn)k_ag_direct_push<16> : (KernelFn)k_ag_direct_push<1>;
    if (pl.algo == A_DIRECT && (pl.variant == 1 || pl.variant == 3) && U != 16) {
      switch (U) {
        case 8: k = (KernelFn)k_ag_direct_push<8>; break;
        case 4: k = (KernelFn)k_ag_direct_push<4>; break;
        case 2: k = (KernelFn)k_ag_direct_push<2>; break;
        default: break;
      }
    }
    if (pl.algo == A_DIRECT && U == 16 && (pl.variant == 2 || pl.variant == 3)) {
      k = pl.variant == 2 ? (KernelFn)k_ag_direct_tma<false> : (KernelFn)k_ag_direct_tma<true>;
      smem = (size_t)w->p_tma_stages * w->p_tma_tile + 8 * (size_t)w->p_tma_stages;
    }
  } else {
    const bool vec = (acc & 15ull) == 0;
    U = vec ? 16 : (int)es;
    int maxp = 2;
    while (maxp < pl.gs) maxp <<= 1;
    k = rs_kernel(pl.dtype, vec, pl.algo, pl.order, maxp, pl.variant);
  }
  if (pl.variant == 6) {  // NVLS: 16-byte vectors through the multicast mapping (caller checked alignment)
    U = 16;
    if (pl.coll == PCCL_ALL_GATHER) k = (KernelFn)k_nvls_ag;
    else if (pl.dtype == PCCL_BFLOAT16) k = (KernelFn)k_nvls_rs<DT_BF16>;
    else if (pl.dtype == PCCL_FLOAT16) k = (KernelFn)k_nvls_rs<DT_F16>;
    else k = (KernelFn)k_nvls_rs<DT_F32>;
  }
  if (!k) return PCCL_ERR_UNSUPPORTED;
  const int64_t epu = U / (int64_t)es > 0 ? U / (int64_t)es : 1;  // elements per unit
  auto units = [&](int64_t e) { return (pl.coll == PCCL_ALL_GATHER) ? e * (int64_t)es / U : e / epu; };
  P.blk = units(pl.blk);
  if (pl.algo == A_DIRECT && pl.variant != 4 && w->p_item_kib > 0) {
    // work-item size in units, a multiple of 32 units (the static slicing grain)
    int64_t it = (w->p_item_kib * 1024 / U) / 32 * 32;
    if (pl.coll != PCCL_ALL_GATHER) it = (w->p_item_kib * 1024 / (int64_t)es / epu) / 32 * 32;
    P.item = std::max<int64_t>(32, it);
  }
  P.sub_stride = units(pl.sub_stride);
  P.istride = units(pl.istride);
  P.send_sub_stride = units(pl.send_sub_stride);
  P.out_sub_stride = units(pl.out_sub_stride);

  // Multi-step protocols hand CTA b's slice of step k to the partner's CTA b
  // at step k + 1, so every rank must cut the same slices: the unit size
  // (from this rank's own buffer alignment in real mode) joins the call
  // signature, and a rank whose buffers are aligned differently raises
  // LengthMismatch everywhere instead of racing. Direct (one-step) kernels
  // only wait on whole CTAs and tolerate it.
  int u_code = 0;
  if (pl.algo != A_DIRECT)
    for (int b = U; b > 1; b >>= 1) ++u_code;
  // ---- rows
  const int nrows = (int)pl.rows.size();
  for (int y = 0; y < nrows; ++y) {
    const Row &rw = pl.rows[y];
    const pccl_comm *g = rw.g;
    P.row_rank[y] = (int8_t)rw.rank;
    int gi = -1;
    for (int m = 0; m < g->gs; ++m) {
      P.gmem[y][m] = (int8_t)g->members[m];
      if (g->members[m] == rw.rank) gi = m;
    }
    P.grank[y] = (int8_t)gi;
    P.base[y] = units(pl.base[rw.rank]);
    P.slot_off[y] = (uint32_t)((size_t)g->slot * PCCL_SLOT_WORDS);
    P.chain_slot_off[y] = pl.chain_slot_off[y];
    P.epoch[y] = 0;  // device-side (CTRL word of the slot), see make_ctx
    P.meta[y] = (hash_meta(pl.coll, pl.algo * 16 + pl.variant, pl.order | (pl.wire << 4) | (u_code << 5), pl.count,
                           pl.dtype, pl.gs) ^
                 (pl.place * 2654435761u) ^
                 w->meta_skew[rw.rank]) & 0x7fffffffu;
  }
  for (int q = 0; q < w->nranks; ++q) {
    P.flags[q] = (uint64_t *)w->segs[0].ptr[q];
    P.send[q] = pl.send[q];
    P.recv[q] = pl.recv[q];
    P.work[q] = pl.work[q];
    P.out[q] = pl.out[q];
  }

  // ---- grid
  const int threads = (int)std::max<int64_t>(64, std::min<int64_t>(w->p_threads, kThreads));
  int ctas = pl.force_ctas > 0 ? pl.force_ctas : (int)w->p_ctas;
  if (ctas <= 0) {
    // auto (measured, tools/sweep.py at p=2/4, profiles/r1_sweep_p*.csv):
    // latency-bound small messages want fewer CTAs (fewer flags); >= 16 MiB
    // wants ~one CTA per SM.
    const double S = (double)pl.gs * (double)pl.count * (double)es;
    ctas = w->emu ? PCCL_MAX_CTAS : (S >= 16.0 * (1 << 20) ? 128 : S >= 4.0 * (1 << 20) ? 64 : 48);
    if (pl.variant == 4) {  // LL: about one 8-byte unit per thread and peer
      const int64_t u = P.blk * (int64_t)pl.nsubblk;
      ctas = (int)std::max<int64_t>(1, std::min<int64_t>(w->emu ? PCCL_MAX_CTAS : 64, (u + threads - 1) / threads));
    }
    if (pl.variant == 8) {  // LL128: one 4-line group per warp and pass
      const int64_t groups = ((P.blk + 14) / 15 + 3) / 4;
      const int64_t wpc = threads / 32;
      ctas = (int)std::max<int64_t>(1, std::min<int64_t>(w->emu ? PCCL_MAX_CTAS : 128, (groups + wpc - 1) / wpc));
    }
  }
  ctas = std::min(ctas, PCCL_MAX_CTAS);
  if (pl.coll == PCCL_REDUCE_SCATTER && pl.variant == 5) ctas = std::max(2, ctas & ~1);  // pusher / folder pairs
  {
    // every CTA must be co-resident (they wait on each other); the occupancy
    // query costs microseconds of host time, so it is cached per configuration
    const OccKey key{(const void *)k, threads, smem};
    int per_sm = -1;
    {
      std::lock_guard<std::mutex> lk(w->occ_mu);  // emulated sub-groups may launch from several threads
      auto it = w->occ_cache.find(key);
      if (it != w->occ_cache.end()) per_sm = it->second;
    }
    if (per_sm < 0) {
      if (smem > 48 * 1024) CK(cudaFuncSetAttribute((const void *)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k, threads, smem));
      std::lock_guard<std::mutex> lk(w->occ_mu);
      w->occ_cache[key] = per_sm;
    }
    const int cap = std::max(1, per_sm) * w->sms;
    ctas = std::max(1, std::min(ctas, cap / nrows));
    if (pl.chain && ctas != pl.force_ctas) return PCCL_ERR_UNSUPPORTED;  // chained slices must match (host checks caps)
  }
  P.ctas = ctas;
  // every flag is per (source, CTA index): the CTA count is part of the call
  // signature (a rank launching another count raises LengthMismatch instead
  // of waiting for CTAs that do not exist until the timeout)
  for (int y = 0; y < nrows; ++y) P.meta[y] = (P.meta[y] ^ ((uint32_t)ctas * 0x9E3779B1u)) & 0x7fffffffu;
  if (pl.variant == 7) {  // recursive halving with per-step work items: ~items_per_cta items per CTA
    const int64_t target = std::min<int64_t>(PCCL_MAX_CTAS, std::max<int64_t>(1, w->p_items_per_cta * ctas));
    const int64_t it = (P.blk + target - 1) / target;
    P.item = std::max<int64_t>(32, (it + 31) / 32 * 32);
  }
  if (w->p_trace) {
    // trace = K: the last K launches, one buffer each (K = 1: memset before
    // every launch; K > 1: consecutive launches run back to back, the ring is
    // cleared once when tracing starts)
    const int K = (int)std::min<int64_t>(w->p_trace, PCCL_TRACE_LAUNCHES);
    const size_t words = (size_t)PCCL_MAXR * PCCL_MAX_CTAS * PCCL_TRACE_EVENTS;
    if (!w->trace_buf) CK(cudaMalloc((void **)&w->trace_buf, words * 8 * PCCL_TRACE_LAUNCHES));
    if (K == 1 || w->trace_seq == 0 || w->trace_rows != nrows || w->trace_ctas != ctas) {
      CK(cudaMemsetAsync(w->trace_buf, 0, words * 8 * (size_t)K, stream));
      w->trace_seq = 0;
    }
    P.trace = w->trace_buf + words * (size_t)(w->trace_seq % K);
    w->trace_seq++;
    w->trace_rows = nrows;
    w->trace_ctas = ctas;
  } else {
    w->trace_seq = 0;
  }
  dim3 grid(ctas, nrows), block(threads);
  if (w->emu) {
    void *args[] = {&P};
    CK(cudaLaunchCooperativeKernel((const void *)k, grid, block, args, smem, stream));
  } else if (w->p_pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k, P));
  } else {
    k<<<grid, block, smem, stream>>>(P);
    CK(cudaGetLastError());
  }
  return PCCL_SUCCESS;
}

// Per-rank buffer binding with staging ------------------------------------
// A buffer peers must read is "symmetric": either it lies in a registered
// segment (then every rank must pass the same segment offset — checked on the
// device through the call signature) or it is copied into the staging
// segment at an SPMD-uniform offset.
struct Binder {
  pccl_world *w;
  cudaStream_t stream;
  size_t cursor = 0;  // staging bump pointer (bytes), SPMD-uniform
  int status = PCCL_SUCCESS;
  uint32_t place = 0;  // hash of symmetric placements (real mode)

  char *stage(int r, size_t bytes, size_t *off_out) {
    size_t off = cursor;
    cursor += align256(bytes);
    if (w->staging < 0 || cursor > w->segs[w->staging].bytes) {
      status = PCCL_ERR_OUT_OF_MEMORY;
      return nullptr;
    }
    *off_out = off;
    return w->segs[w->staging].ptr[r] + off;
  }
  void fill(int r, int seg, size_t off, char **per, char *own) {
    for (int q = 0; q < w->nranks; ++q) {
      if (w->emu && q != r) continue;  // emulation: each row binds its own rank only
      per[q] = w->segs[seg].ptr[q] ? w->segs[seg].ptr[q] + off : nullptr;
    }
    per[r] = own;
  }
  // Returns false on error. *staged = local staging alias when copied.
  bool symmetric(int r, const void *user, size_t bytes, bool copy_in, char **per, char **staged) {
    int seg;
    size_t off;
    if (staged) *staged = nullptr;
    if (bytes == 0) {
      per[r] = (char *)user;
      return true;
    }
    if (resolve(w, r, user, bytes, &seg, &off)) {
      fill(r, seg, off, per, (char *)user);
      place = place * 31u + (uint32_t)seg * 7919u + (uint32_t)(off >> 8) + 1u;
      return true;
    }
    size_t soff;
    char *p = stage(r, bytes, &soff);
    if (!p) return false;
    fill(r, w->staging, soff, per, p);
    place = place * 31u + 17u;
    w->p_staged_bytes += (int64_t)bytes;  // staging copy in or out: the buffer was not registered
    if (copy_in && cudaMemcpyAsync(p, user, bytes, cudaMemcpyDeviceToDevice, stream) != cudaSuccess) {
      status = PCCL_ERR_CUDA;
      return false;
    }
    if (staged) *staged = p;
    return true;
  }
  // Internal symmetric scratch (same staging offset on every rank).
  bool scratch(int r, size_t bytes, char **per) {
    size_t soff;
    char *p = stage(r, bytes, &soff);
    if (!p) return false;
    fill(r, w->staging, soff, per, p);
    return true;
  }
};

// LL protocol choice (device.cuh): small direct collectives whose per-peer
// message fits an LL region. Depends only on SPMD-uniform values (size,
// world parameters), never on this rank's pointers, so all members agree.
// Auto threshold (tools/latency.py, p=2/4, graph-replayed, r1): LL beats the
// flag protocol until a rank's total LL egress reaches ~0.75-1 MiB (p=2: 9.4
// vs 11.2 us at 1 MiB per peer; p=4: tie at 256 KiB per peer).
constexpr size_t kLLEgress = 768u << 10;
bool use_ll(const pccl_world *w, int64_t variant_param, size_t msg_bytes, int gs) {
  if (variant_param != -1 && variant_param != 4) return false;
  size_t cap = PCCL_LL_MAX_PAYLOAD;
  if (variant_param != 4) {
    const size_t lim = w->p_ll_max < 0 ? kLLEgress / (size_t)std::max(1, gs - 1) : (size_t)w->p_ll_max;
    cap = std::min(cap, lim);
  }
  return gs <= PCCL_MAXR && msg_bytes > 0 && msg_bytes % 8 == 0 && msg_bytes <= cap;
}

// LL128 (direct collectives): requested (variant 8) or automatic for
// messages above the LL range up to `ll128_max` payload bytes per peer; a
// message must fit one region (PCCL_LL128_MAX_PAYLOAD). SPMD-uniform inputs
// only, like use_ll.
// A reduce-scatter's owner folds p - 1 line streams: measured (tools/tune.py,
// bf16) it wins up to ~3 MiB of egress per rank (p=4: 1 MiB per peer +2..10 %,
// 1.25 MiB -4 %; p=2 up to the region, +23..31 %), so its automatic range is
// also capped by kLL128RsEgress / (p - 1). All-gathers were measured up to
// 5.25 MiB of egress (p=4, 7 MiB: +4 %); beyond that (p=8 with full regions)
// they are capped at kLL128AgEgress / (p - 1), unmeasured above.
constexpr size_t kLL128RsEgress = (size_t)3 << 20;
constexpr size_t kLL128AgEgress = (size_t)6 << 20;
bool use_ll128(const pccl_world *w, int64_t v, size_t msg_bytes, int gs, bool reduce) {
  size_t cap = PCCL_LL128_MAX_PAYLOAD;
  if (v == -1) {
    if (w->p_ll128_max <= 0) return false;
    cap = std::min(cap, (size_t)w->p_ll128_max);
    cap = std::min(cap, (reduce ? kLL128RsEgress : kLL128AgEgress) / (size_t)std::max(1, gs - 1));
  } else if (v != 8) {
    return false;
  }
  return gs <= PCCL_MAXR && msg_bytes > 0 && msg_bytes % 8 == 0 && msg_bytes <= cap;
}

// LL kernels touch user buffers only locally, with 8-byte accesses: a
// misaligned buffer on this rank is bounced through local staging.
bool ll_local(Binder &B, int r, char *&p, size_t bytes, bool copy_in, std::vector<std::pair<char *, char *>> *out) {
  if (((uintptr_t)p & 7u) == 0) return true;
  size_t off;
  char *s = B.stage(r, bytes, &off);
  if (!s) return false;
  if (copy_in && cudaMemcpyAsync(s, p, bytes, cudaMemcpyDeviceToDevice, B.stream) != cudaSuccess) {
    B.status = PCCL_ERR_CUDA;
    return false;
  }
  if (out) out->push_back({s, p});
  p = s;
  return true;
}

// A device-reported error poisons the world: kernels that aborted did not
// finish their protocol, so every later call fails fast with the same code
// until pccl_world_reset_flags (emulation) or the world is recreated.
int check_world_err(pccl_world *w) {
  const int e = *w->err_host;
  if (e && !w->poisoned) w->poisoned = e;
  return w->poisoned;
}

// --------------------------------------------------------------------------
// Copy-engine all-gather (ag_variant 5, real mode, ring / recursive doubling).
// tools/probe.py measured the copy engines at 737 GB/s per direction for a
// pairwise exchange against 680 (SM stores) / 640 (SM loads), and both
// all-gather schedules that exchange pairwise are pure copies. Each step is
// one cudaMemcpyAsync from my recv into the partner's symmetric recv; the
// cross-GPU handshakes are stream memory operations on the META words of the
// group's flag slot (unused by the kernels): cuStreamWriteValue64 into the
// reader's arena (it carries a system-scope fence after the copy before it)
// and cuStreamWaitValue64 (>=) on my own arena. Values are a per-group host
// counter; the path is never taken while the stream is being captured, so
// the count stays exact. No kernel runs and the device epoch is untouched.
// --------------------------------------------------------------------------
struct MemOps {
  bool ok = false;
  CUresult (*wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
  CUresult (*write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
};

MemOps &memops(int device) {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [&] {
    void *fw = nullptr, *fr = nullptr, *fa = nullptr;
    cudaDriverEntryPointQueryResult q1, q2, q3;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &fw, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWriteValue64", &fr, cudaEnableDefault, &q2) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fa, cudaEnableDefault, &q3) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || q3 != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return;
    }
    int v = 0;
    auto attr = (CUresult(*)(int *, CUdevice_attribute, CUdevice))fa;
    if (attr(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, (CUdevice)device) != CUDA_SUCCESS) v = 0;
    m.wait64 = (CUresult(*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int))fw;
    m.write64 = (CUresult(*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int))fr;
    m.ok = v != 0;
  });
  return m;
}

// META word `idx` that member `src` writes into world rank q's arena
CUdeviceptr ce_flag(const pccl_comm *c, int q, int src, int idx) {
  uint64_t *slot = (uint64_t *)c->w->segs[0].ptr[q] + (size_t)c->slot * PCCL_SLOT_WORDS;
  return (CUdeviceptr)(slot + ((size_t)(F_META * PCCL_MAXR + src) * PCCL_MAX_CTAS + idx));
}

// The path is explicitly requested (ag_variant 5) and must be taken by every
// member: a call that does not qualify on this rank fails with Unsupported
// instead of silently falling back to kernels (a member that took the other
// path would wait for this one until the timeout, not forever: the waits are
// k_ce_wait kernels bounded by the world timeout, which flood ABORT on expiry).
int ce_all_gather(pccl_comm *c, int algo, const void *send, void *recv, size_t blk, cudaStream_t s) {
  pccl_world *w = c->w;
  if (w->emu) return PCCL_ERR_UNSUPPORTED;
  if (blk == 0) return PCCL_SUCCESS;
  MemOps &mo = memops(w->device);
  if (!mo.ok) return PCCL_ERR_UNSUPPORTED;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return PCCL_ERR_UNSUPPORTED;
  }
  const int gs = c->gs, gi = c->gi, me = w->rank;
  int seg;
  size_t off;
  if (gi < 0 || !resolve(w, me, recv, gs * blk, &seg, &off)) return PCCL_ERR_UNSUPPORTED;  // peers write into my recv
  auto peer_recv = [&](int m) { return w->segs[seg].ptr[c->members[m]] + off; };
  char *my = (char *)recv;
  const uint64_t e = ++w->ce_calls[c->slot];
  CUstream cs = (CUstream)s;
  CeWait W;
  memset(&W, 0, sizeof(W));
  W.target = e;
  W.err = w->err_dev;
  W.mirror = (uint64_t *)w->segs[0].ptr[me] + PCCL_WCTRL_OFF + PCCL_WCTRL_ERR;
  W.timeout_ns = w->p_timeout_ms * 1000000ll;
  W.gs = gs;
  for (int m = 0; m < gs; ++m)
    W.meta[m] = (uint64_t *)c->w->segs[0].ptr[c->members[m]] + (size_t)c->slot * PCCL_SLOT_WORDS +
                (size_t)F_META * PCCL_MAXR * PCCL_MAX_CTAS;
  auto wait = [&](int src, int idx) -> int {
    W.word = (const uint64_t *)ce_flag(c, me, src, idx);
    k_ce_wait<<<1, 128, 0, s>>>(W);
    return cuda_err(cudaGetLastError());
  };
#define CE(x)                                        \
  do {                                               \
    if ((x) != CUDA_SUCCESS) return PCCL_ERR_CUDA;   \
  } while (0)
#define CW(x)                \
  do {                       \
    const int st_ = (x);     \
    if (st_) return st_;     \
  } while (0)
  if ((const char *)send != my + (size_t)gi * blk)
    CK(cudaMemcpyAsync(my + (size_t)gi * blk, send, blk, cudaMemcpyDeviceToDevice, s));
  if (algo == A_REC) {
    const int L = 31 - __builtin_clz(gs);
    for (int k = 0; k < L; ++k)  // my recv may be written (every partner writes into it)
      CE(mo.write64(cs, ce_flag(c, c->members[gi ^ (1 << k)], gi, 0), e, 0));
    for (int k = 0; k < L; ++k) {
      const int partner = gi ^ (1 << k), start = (gi >> k) << k;
      CW(wait(partner, 0));
      if (k > 0) CW(wait(gi ^ (1 << (k - 1)), k));
      CK(cudaMemcpyAsync(peer_recv(partner) + (size_t)start * blk, my + (size_t)start * blk, ((size_t)1 << k) * blk,
                         cudaMemcpyDeviceToDevice, s));
      CE(mo.write64(cs, ce_flag(c, c->members[partner], gi, k + 1), e, 0));
    }
    CW(wait(gi ^ (1 << (L - 1)), L));
  } else {  // ring: step t forwards block (gi - t + 1) to next (collectives.py:70-75)
    const int next = (gi + 1) % gs, prev = (gi + gs - 1) % gs;
    CE(mo.write64(cs, ce_flag(c, c->members[prev], gi, 0), e, 0));
    CW(wait(next, 0));
    for (int t = 1; t < gs; ++t) {
      if (t > 1) CW(wait(prev, t - 1));
      const int b = (gi - t + 1 + gs) % gs;
      CK(cudaMemcpyAsync(peer_recv(next) + (size_t)b * blk, my + (size_t)b * blk, blk, cudaMemcpyDeviceToDevice, s));
      CE(mo.write64(cs, ce_flag(c, c->members[next], gi, t), e, 0));
    }
    CW(wait(prev, gs - 1));
  }
#undef CE
#undef CW
  return PCCL_SUCCESS;
}

// --------------------------------------------------------------------------
// NVLS multicast segments (driver VMM + multicast API through cudart's entry
// points, so the library has no link-time dependency on libcuda).
// --------------------------------------------------------------------------
struct DrvNvls {
  bool ok = false;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
  CUresult (*mcGran)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
  CUresult (*mcAddDev)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*mcBind)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                     unsigned long long);
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*exportH)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
  CUresult (*importH)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType);
  CUresult (*memCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
  CUresult (*memRelease)(CUmemGenericAllocationHandle);
  CUresult (*reserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*addrFree)(CUdeviceptr, size_t);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
  CUresult (*attr)(int *, CUdevice_attribute, CUdevice);
};

DrvNvls &drv_nvls() {
  static DrvNvls d;
  static std::once_flag once;
  std::call_once(once, [&] {
    bool ok = true;
    auto get = [&](const char *name, auto &fn) {
      void *f = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
          !f) {
        cudaGetLastError();
        ok = false;
        return;
      }
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(f);
    };
    get("cuMulticastCreate", d.mcCreate);
    get("cuMulticastGetGranularity", d.mcGran);
    get("cuMulticastAddDevice", d.mcAddDev);
    get("cuMulticastBindMem", d.mcBind);
    get("cuMulticastUnbind", d.mcUnbind);
    get("cuMemExportToShareableHandle", d.exportH);
    get("cuMemImportFromShareableHandle", d.importH);
    get("cuMemCreate", d.memCreate);
    get("cuMemRelease", d.memRelease);
    get("cuMemAddressReserve", d.reserve);
    get("cuMemAddressFree", d.addrFree);
    get("cuMemMap", d.map);
    get("cuMemUnmap", d.unmap);
    get("cuMemSetAccess", d.setAccess);
    get("cuDeviceGetAttribute", d.attr);
    d.ok = ok;
  });
  return d;
}

CUmulticastObjectProp nvls_prop(const pccl_world *w, size_t bytes) {
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)w->nranks;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  return mp;
}

// --------------------------------------------------------------------------
// flat collectives (shared by real and emulation mode)
// --------------------------------------------------------------------------
// ranks: world ranks this process executes (real: {me}; emulation: all members)
int do_all_gather(pccl_comm *c, int algo, const std::vector<int> &ranks, const void *const *sends,
                  void *const *recvs, size_t count, int dtype, cudaStream_t stream) {
  pccl_world *w = c->w;
  const size_t es = dt_size(dtype);
  if (!es) return PCCL_ERR_INVALID_ARGUMENT;
  if (algo < 0 || algo > 2) return PCCL_ERR_INVALID_ARGUMENT;
  if (algo == A_REC && !is_pow2(c->gs)) return PCCL_ERR_NON_POWER_OF_TWO;
  CK(cudaSetDevice(w->device));
  const int gs = c->gs;
  const size_t blk_bytes = count * es;
  if (gs == 1) {  // collectives.py:66-67
    for (size_t i = 0; i < ranks.size(); ++i)
      if (blk_bytes && sends[i] != recvs[i])
        CK(cudaMemcpyAsync(recvs[i], sends[i], blk_bytes, cudaMemcpyDeviceToDevice, stream));
    return PCCL_SUCCESS;
  }
  Plan pl;
  pl.coll = PCCL_ALL_GATHER;
  pl.algo = algo;
  pl.dtype = dtype;
  pl.count = count;
  pl.gs = gs;
  pl.blk = (int64_t)count;
  pl.istride = (int64_t)count;
  pl.send_sub_stride = (int64_t)count;
  const bool ll = algo == A_DIRECT && use_ll(w, w->p_ag_variant, blk_bytes, gs);
  if (algo == A_DIRECT && (ll || use_ll128(w, w->p_ag_variant, blk_bytes, gs, false))) {
    pl.variant = ll ? 4 : 8;
    pl.local_copy = 0;  // OR over the rows below: one value per launch, a self-copy is harmless
    Binder B{w, stream};
    std::vector<std::pair<char *, char *>> copy_out;
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i];
      int gi = -1;
      for (int m = 0; m < gs; ++m)
        if (c->members[m] == r) gi = m;
      if (gi < 0) return PCCL_ERR_INDEX_OUT_OF_RANGE;
      pl.rows.push_back({r, c});
      B.cursor = 0;
      char *snd = (char *)sends[i], *rcv = (char *)recvs[i];
      const bool inplace = snd == rcv + (size_t)gi * blk_bytes;
      if (!ll_local(B, r, rcv, gs * blk_bytes, false, &copy_out)) return B.status;
      if (inplace) snd = rcv + (size_t)gi * blk_bytes;
      if (!ll_local(B, r, snd, blk_bytes, true, nullptr)) return B.status;
      pl.send[r] = snd;
      pl.recv[r] = rcv;
      pl.local_copy |= snd != rcv + (size_t)gi * blk_bytes;  // any row (a self-copy is harmless)
    }
    int s = launch(w, pl, stream);
    if (s) return s;
    for (auto &co : copy_out) CK(cudaMemcpyAsync(co.second, co.first, gs * blk_bytes, cudaMemcpyDeviceToDevice, stream));
    return PCCL_SUCCESS;
  }
  if (w->p_ag_variant == 5 && !w->emu && algo != A_DIRECT) return ce_all_gather(c, algo, sends[0], recvs[0], blk_bytes, stream);
  {
    // Data movement. auto: push (posted NVLink stores, saturates the links
    // with few SMs) whenever the output is symmetric; a direct all-gather into
    // an unregistered output pulls instead (only the small send is staged).
    int v = (int)w->p_ag_variant;
    if (v == 4 || v == 5 || v == 8) v = -1;  // LL / copy engine / LL128 requested but this call does not qualify
    if (v < 0) {
      int seg;
      size_t off;
      const bool recv_reg = resolve(w, ranks[0], recvs[0], gs * blk_bytes, &seg, &off);
      v = (recv_reg || algo != A_DIRECT) ? 1 : 0;
    }
    if (algo != A_DIRECT && v != 1) v = 0;  // TMA variants exist for direct only
    pl.variant = v;
    pl.rank_final = 1;  // flat call: every rank takes the same choice
  }
  Binder B{w, stream};
  std::vector<std::pair<char *, char *>> copy_out;  // (staged recv, user recv)
  pl.local_copy = 0;  // OR over the rows below: one value per launch, a self-copy is harmless
  for (size_t i = 0; i < ranks.size(); ++i) {
    const int r = ranks[i];
    int gi = -1;
    for (int m = 0; m < gs; ++m)
      if (c->members[m] == r) gi = m;
    if (gi < 0) return PCCL_ERR_INDEX_OUT_OF_RANGE;
    pl.rows.push_back({r, c});
    B.cursor = 0;
    if (algo == A_DIRECT && (pl.variant == 1 || pl.variant == 3)) {
      // push: I write into my peers' recv; send is read locally only
      char *staged = nullptr;
      if (!B.symmetric(r, recvs[i], gs * blk_bytes, false, pl.recv, &staged)) return B.status;
      if (staged) copy_out.push_back({staged, (char *)recvs[i]});
      pl.send[r] = (char *)sends[i];
      pl.local_copy |= staged || sends[i] != (const char *)recvs[i] + (size_t)gi * blk_bytes;
    } else if (algo == A_DIRECT) {
      // peers read my send; my recv is written locally only
      if (!B.symmetric(r, sends[i], blk_bytes, true, pl.send, nullptr)) return B.status;
      pl.recv[r] = (char *)recvs[i];
      pl.local_copy |= sends[i] != (const char *)recvs[i] + (size_t)gi * blk_bytes;
    } else {
      // peers forward out of my recv; send is read locally only
      char *staged = nullptr;
      if (!B.symmetric(r, recvs[i], gs * blk_bytes, false, pl.recv, &staged)) return B.status;
      if (staged) copy_out.push_back({staged, (char *)recvs[i]});
      pl.send[r] = (char *)sends[i];
      pl.local_copy |= staged || sends[i] != (const char *)recvs[i] + (size_t)gi * blk_bytes;
    }
  }
  pl.place = w->emu ? 0 : B.place;
  int s = launch(w, pl, stream);
  if (s) return s;
  for (auto &co : copy_out) CK(cudaMemcpyAsync(co.second, co.first, gs * blk_bytes, cudaMemcpyDeviceToDevice, stream));
  return PCCL_SUCCESS;
}

int do_reduce_scatter(pccl_comm *c, int algo, int order, const std::vector<int> &ranks, const void *const *sends,
                      void *const *recvs, size_t recvcount, int dtype, cudaStream_t stream) {
  pccl_world *w = c->w;
  if (dtype != PCCL_FLOAT32 && dtype != PCCL_BFLOAT16 && dtype != PCCL_FLOAT16) return PCCL_ERR_UNSUPPORTED;
  // order | PCCL_ORDER_WIRE (direct only): round the partial after every add,
  // exactly where ring / recursive halving store theirs
  const int wire = (order & PCCL_ORDER_WIRE) ? 1 : 0;
  order &= ~PCCL_ORDER_WIRE;
  if (algo < 0 || algo > 2 || order < 0 || order > 2) return PCCL_ERR_INVALID_ARGUMENT;
  const int gs = c->gs;
  if (algo == A_REC && !is_pow2(gs)) return PCCL_ERR_NON_POWER_OF_TWO;
  if (algo == A_DIRECT && order == O_REC && !is_pow2(gs)) return PCCL_ERR_NON_POWER_OF_TWO;
  CK(cudaSetDevice(w->device));
  const size_t es = dt_size(dtype);
  const size_t chunk_bytes = recvcount * es;
  if (gs == 1) {  // collectives.py:88-89
    for (size_t i = 0; i < ranks.size(); ++i)
      if (chunk_bytes && sends[i] != recvs[i])
        CK(cudaMemcpyAsync(recvs[i], sends[i], chunk_bytes, cudaMemcpyDeviceToDevice, stream));
    return PCCL_SUCCESS;
  }
  Plan pl;
  pl.coll = PCCL_REDUCE_SCATTER;
  pl.algo = algo;
  pl.order = algo == A_DIRECT ? order : 0;
  pl.wire = algo == A_DIRECT ? wire : 0;
  pl.dtype = dtype;
  pl.count = recvcount;
  pl.gs = gs;
  pl.blk = (int64_t)recvcount;
  pl.istride = (int64_t)recvcount;
  pl.out_sub_stride = (int64_t)recvcount;
  const bool ll = algo == A_DIRECT && use_ll(w, w->p_rs_variant, chunk_bytes, gs);
  if (algo == A_DIRECT && (ll || use_ll128(w, w->p_rs_variant, chunk_bytes, gs, true))) {
    pl.variant = ll ? 4 : 8;
    pl.local_copy = 0;  // OR over the rows below: one value per launch, a self-copy is harmless
    Binder B{w, stream};
    std::vector<std::pair<char *, char *>> copy_out;
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i];
      bool member = false;
      for (int m = 0; m < gs; ++m) member |= c->members[m] == r;
      if (!member) return PCCL_ERR_INDEX_OUT_OF_RANGE;
      pl.rows.push_back({r, c});
      B.cursor = 0;
      char *snd = (char *)sends[i], *rcv = (char *)recvs[i];
      if (!ll_local(B, r, snd, gs * chunk_bytes, true, nullptr)) return B.status;
      if (!ll_local(B, r, rcv, chunk_bytes, false, &copy_out)) return B.status;
      pl.send[r] = snd;
      pl.out[r] = rcv;
    }
    int s = launch(w, pl, stream);
    if (s) return s;
    for (auto &co : copy_out) CK(cudaMemcpyAsync(co.second, co.first, chunk_bytes, cudaMemcpyDeviceToDevice, stream));
    return PCCL_SUCCESS;
  }
  {
    // auto: pull (peer loads fused with the add, no staging hop) for every
    // algorithm when the input is symmetric; push when it is unregistered (no
    // input staging copy). The ring's push variant ends with a purely local
    // step (carry + own chunk -> output) that leaves NVLink idle in the tail:
    // pull ring measured 580 vs 502 GB/s at p=2 and 597 vs 583 at p=4
    // (128 MiB bf16, profiles/r2_rs_ring_pull_vs_push.txt).
    int v = (int)w->p_rs_variant;
    if (v == 4 || v == 8) v = -1;  // LL / LL128 requested but this message does not qualify
    if (v < 0) {
      int seg;
      size_t off;
      const bool send_reg = resolve(w, ranks[0], sends[0], gs * chunk_bytes, &seg, &off);
      v = !send_reg ? 1 : 0;
    }
    pl.variant = v == 1 ? 1 : (v == 5 && algo == A_DIRECT) ? 5 : (v == 7 && algo == A_REC) ? 7 : 0;
  }
  Binder B{w, stream};
  for (size_t i = 0; i < ranks.size(); ++i) {
    const int r = ranks[i];
    bool member = false;
    for (int m = 0; m < gs; ++m) member |= c->members[m] == r;
    if (!member) return PCCL_ERR_INDEX_OUT_OF_RANGE;
    pl.rows.push_back({r, c});
    B.cursor = 0;
    if (pl.variant == 1 || pl.variant == 5) {
      // push: send is read locally only; peers write into my staging (recv)
      pl.send[r] = (char *)sends[i];
      if (!B.scratch(r, gs * chunk_bytes, pl.recv)) return B.status;
      if (algo == A_REC && !B.scratch(r, gs * chunk_bytes, pl.work)) return B.status;
      pl.out[r] = (char *)recvs[i];
      continue;
    }
    if (!B.symmetric(r, sends[i], gs * chunk_bytes, true, pl.send, nullptr)) return B.status;
    if (algo != A_DIRECT) {
      B.cursor = align256(gs * chunk_bytes);  // work at the same offset on every rank
      if (!B.scratch(r, gs * chunk_bytes, pl.work)) return B.status;
    }
    pl.out[r] = (char *)recvs[i];
  }
  pl.place = w->emu ? 0 : B.place;
  return launch(w, pl, stream);
}

std::vector<int> one(int r) { return std::vector<int>{r}; }

pccl_comm *cached_group(pccl_world *w, const std::vector<int> &members, int comm_id) {
  uint32_t mask = 0;
  for (int m : members) mask |= 1u << m;
  const uint32_t key = mask;  // one cached object per member set (order checked below)
  auto it = w->comm_cache.find(key);
  if (it != w->comm_cache.end()) {
    bool same = it->second->gs == (int)members.size();
    for (size_t i = 0; same && i < members.size(); ++i) same = it->second->members[i] == members[i];
    if (same) return it->second;
  }
  pccl_comm *c = nullptr;
  if (pccl_comm_create(w, members.data(), (int)members.size(), comm_id, &c) != PCCL_SUCCESS) return nullptr;
  if (it != w->comm_cache.end()) pccl_comm_destroy(it->second);
  w->comm_cache[key] = c;
  return c;
}

// --------------------------------------------------------------------------
// hierarchical (hierarchy.py:158-195) over a communicator `mem` (topology rank
// g -> world rank mem[g]; the world communicator is mem = 0..p-1); virtual
// nodes n = g / M, local j = g % M
// --------------------------------------------------------------------------
bool topo_index(const pccl_world *w, const std::vector<int> &mem, int *topo) {
  for (int q = 0; q < PCCL_MAXR; ++q) topo[q] = -1;
  for (size_t g = 0; g < mem.size(); ++g) {
    if (mem[g] < 0 || mem[g] >= w->nranks || topo[mem[g]] >= 0) return false;
    topo[mem[g]] = (int)g;
  }
  return true;
}
std::vector<int> iota_ranks(int n) {
  std::vector<int> v(n);
  for (int i = 0; i < n; ++i) v[i] = i;
  return v;
}

int do_hier_all_gather(pccl_world *w, const std::vector<int> &mem, int N, int M, int inter, const std::vector<int> &ranks,
                       const void *const *sends, void *const *recvs, size_t count, int dtype, cudaStream_t stream) {
  if (N < 1 || M < 1 || N * M != (int)mem.size()) return PCCL_ERR_LENGTH_MISMATCH;
  int topo[PCCL_MAXR];  // world rank -> topology rank g (index in mem)
  if (!topo_index(w, mem, topo)) return PCCL_ERR_INVALID_ARGUMENT;
  if (inter != A_RING && inter != A_REC) return PCCL_ERR_INVALID_ARGUMENT;
  if (inter == A_REC && !is_pow2(N)) return PCCL_ERR_NON_POWER_OF_TWO;
  const size_t es = dt_size(dtype);
  if (!es) return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  const int p = N * M;
  const size_t out_bytes = (size_t)p * count * es;
  // symmetric output (both phases forward out of it)
  Binder B{w, stream};
  char *outp[PCCL_MAXR] = {};
  std::vector<std::pair<char *, char *>> copy_out;
  for (size_t i = 0; i < ranks.size(); ++i) {
    const int r = ranks[i];
    B.cursor = 0;
    char *staged = nullptr;
    if (!B.symmetric(r, recvs[i], out_bytes, false, outp, &staged)) return B.status;
    if (staged) copy_out.push_back({staged, (char *)recvs[i]});
  }
  const uint32_t place = w->emu ? 0 : B.place;
  // Chain the two phases (device.cuh "chained launches") when both exist, the
  // slices of both launches are identical (16-byte units everywhere, static
  // slices, the same CTA count) and PDL is on.
  // The CTA count is fixed by SPMD-uniform conditions only; whether the two
  // launches are chained also depends on this rank's pointers, which only
  // changes local sequencing.
  const bool uniform = !w->emu && w->p_pdl && w->p_hier_chain && N > 1 && M > 1 && w->p_item_kib == 0 &&
                       w->p_ctas <= 128 && (count * es) % 16 == 0;
  bool chain = uniform;
  for (size_t i = 0; chain && i < ranks.size(); ++i)
    chain = ((uintptr_t)outp[ranks[i]] % 16 == 0) && ((uintptr_t)sends[i] % 16 == 0);
  const int chain_ctas = w->p_ctas > 0 ? (int)w->p_ctas : 128;
  // phase 1: inter-node all-gather on every stride-M group, blocks land at
  // their global positions (g*count) directly (fused shuffle)
  if (N > 1) {
    Plan pl;
    if (uniform) pl.force_ctas = chain_ctas;
    if (chain) {
      pl.chain = 1;
      for (size_t i = 0; i < ranks.size(); ++i) {  // row i: the intra group of ranks[i] runs phase 2
        const int nd = topo[ranks[i]] / M;
        std::vector<int> grp;
        for (int l = 0; l < M; ++l) grp.push_back(mem[nd * M + l]);
        pccl_comm *g2 = cached_group(w, grp, 1 + M + nd);
        if (!g2) return PCCL_ERR_CUDA;
        pl.chain_slot_off[i] = (uint32_t)((size_t)g2->slot * PCCL_SLOT_WORDS);
      }
    }
    pl.coll = PCCL_ALL_GATHER; pl.algo = inter; pl.dtype = dtype; pl.count = count; pl.gs = N;
    pl.blk = (int64_t)count; pl.istride = (int64_t)M * count; pl.send_sub_stride = (int64_t)count;
    pl.local_copy = 1;
    pl.place = place;
    pl.variant = w->p_ag_variant == 0 ? 0 : 1;  // push (recv is symmetric)
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i], j = topo[r] % M;
      std::vector<int> grp;
      for (int n = 0; n < N; ++n) grp.push_back(mem[n * M + j]);
      pccl_comm *g = cached_group(w, grp, 1 + j);
      if (!g) return PCCL_ERR_CUDA;
      pl.rows.push_back({r, g});
      pl.base[r] = (int64_t)j * count;
      pl.send[r] = (char *)sends[i];
    }
    for (int g = 0; g < N * M; ++g) { const int q = mem[g]; pl.recv[q] = outp[q]; pl.base[q] = (int64_t)(g % M) * count; }
    int s = launch(w, pl, stream);
    if (s) return s;
  } else {
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i];
      if (count) CK(cudaMemcpyAsync(outp[r] + (size_t)topo[r] * count * es, sends[i], count * es, cudaMemcpyDeviceToDevice, stream));
    }
  }
  // phase 2: intra-node all-gather; member l's block = N sub-blocks at
  // (n*M + l)*count. The reference's intra phase is a ring (hierarchy.py:171);
  // an all-gather's output does not depend on the schedule, so for M >= 3 the
  // one-step direct push replaces the M - 1 ring steps (param "hier_intra":
  // -1 auto, 0 ring, 1 direct).
  if (M > 1) {
    Plan pl;
    const bool direct = w->p_hier_intra == 1 || (w->p_hier_intra < 0 && M >= 3);
    pl.coll = PCCL_ALL_GATHER; pl.algo = direct ? A_DIRECT : A_RING; pl.dtype = dtype; pl.count = (size_t)N * count;
    pl.gs = M;
    if (uniform) pl.force_ctas = chain_ctas;
    if (chain) pl.chain = 2;
    pl.nsubblk = N; pl.blk = (int64_t)count; pl.sub_stride = (int64_t)M * count; pl.istride = (int64_t)count;
    pl.send_sub_stride = (int64_t)count; pl.local_copy = 0; pl.place = place;
    pl.variant = w->p_ag_variant == 0 ? 0 : 1;
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i], n = topo[r] / M;
      std::vector<int> grp;
      for (int l = 0; l < M; ++l) grp.push_back(mem[n * M + l]);
      pccl_comm *g = cached_group(w, grp, 1 + M + n);
      if (!g) return PCCL_ERR_CUDA;
      pl.rows.push_back({r, g});
    }
    for (int g = 0; g < N * M; ++g) {
      const int q = mem[g];
      pl.recv[q] = outp[q];
      // ring forwards out of recv; direct reads my block (N sub-blocks at
      // stride M * count, starting at local rank * count) as its send
      pl.send[q] = direct ? outp[q] + (size_t)(g % M) * count * es : outp[q];
    }
    if (direct) pl.send_sub_stride = (int64_t)M * count;
    int s = launch(w, pl, stream);
    if (s) return s;
  }
  for (auto &co : copy_out) CK(cudaMemcpyAsync(co.second, co.first, out_bytes, cudaMemcpyDeviceToDevice, stream));
  return PCCL_SUCCESS;
}

int do_hier_reduce_scatter(pccl_world *w, const std::vector<int> &mem, int N, int M, int inter, const std::vector<int> &ranks,
                           const void *const *sends, void *const *recvs, size_t n, int dtype, cudaStream_t stream) {
  if (N < 1 || M < 1 || N * M != (int)mem.size()) return PCCL_ERR_LENGTH_MISMATCH;
  int topo[PCCL_MAXR];  // world rank -> topology rank g (index in mem)
  if (!topo_index(w, mem, topo)) return PCCL_ERR_INVALID_ARGUMENT;
  if (inter != A_RING && inter != A_REC) return PCCL_ERR_INVALID_ARGUMENT;
  if (inter == A_REC && !is_pow2(N)) return PCCL_ERR_NON_POWER_OF_TWO;
  if (dtype != PCCL_FLOAT32 && dtype != PCCL_BFLOAT16 && dtype != PCCL_FLOAT16) return PCCL_ERR_UNSUPPORTED;
  CK(cudaSetDevice(w->device));
  const size_t es = dt_size(dtype);
  const int p = N * M;
  const size_t in_bytes = (size_t)p * n * es, part_bytes = (size_t)N * n * es;
  Binder B{w, stream};
  char *sendp[PCCL_MAXR] = {}, *work[PCCL_MAXR] = {}, *part[PCCL_MAXR] = {}, *work2[PCCL_MAXR] = {};
  for (size_t i = 0; i < ranks.size(); ++i) {
    const int r = ranks[i];
    B.cursor = 0;
    if (!B.symmetric(r, sends[i], in_bytes, true, sendp, nullptr)) return B.status;
    B.cursor = align256(in_bytes);
    if (!B.scratch(r, in_bytes, work) || !B.scratch(r, part_bytes, part) || !B.scratch(r, part_bytes, work2))
      return B.status;
  }
  const uint32_t place = w->emu ? 0 : B.place;
  // chained phases (see do_hier_all_gather)
  // (CTA count from SPMD-uniform conditions only, see do_hier_all_gather)
  const bool uniform = !w->emu && w->p_pdl && w->p_hier_chain && N > 1 && M > 1 && w->p_item_kib == 0 &&
                       w->p_ctas <= 128 && (n * es) % 16 == 0 && w->p_rs_variant != 1;
  bool chain = uniform;
  for (size_t i = 0; chain && i < ranks.size(); ++i)
    chain = ((uintptr_t)sendp[ranks[i]] % 16 == 0) && ((uintptr_t)recvs[i] % 16 == 0);
  const int chain_ctas = w->p_ctas > 0 ? (int)w->p_ctas : 128;
  // phase 1: intra reduce-scatter; chunk l = N sub-blocks {nd*M + l}. The
  // reference's ring (hierarchy.py:193) fixes the add order (left fold from
  // l+1) and, in bf16 / fp16, a rounding after every add; for M >= 3 the
  // one-step direct kernel folds in exactly that order with the same rounding
  // points (wire) — bit-identical, M - 2 fewer steps (param "hier_intra").
  if (M > 1) {
    Plan pl;
    const bool direct = w->p_hier_intra == 1 || (w->p_hier_intra < 0 && M >= 3);
    pl.coll = PCCL_REDUCE_SCATTER; pl.algo = direct ? A_DIRECT : A_RING; pl.dtype = dtype; pl.count = (size_t)N * n;
    pl.gs = M;
    pl.order = O_RING;
    pl.wire = 1;
    if (uniform) pl.force_ctas = chain_ctas;
    if (chain) {
      pl.chain = 1;
      for (size_t i = 0; i < ranks.size(); ++i) {  // row i: the inter group of ranks[i] runs phase 2
        const int j = topo[ranks[i]] % M;
        std::vector<int> grp;
        for (int nd = 0; nd < N; ++nd) grp.push_back(mem[nd * M + j]);
        pccl_comm *g2 = cached_group(w, grp, 1 + j);
        if (!g2) return PCCL_ERR_CUDA;
        pl.chain_slot_off[i] = (uint32_t)((size_t)g2->slot * PCCL_SLOT_WORDS);
      }
    }
    pl.nsubblk = N; pl.blk = (int64_t)n; pl.sub_stride = (int64_t)M * n; pl.istride = (int64_t)n;
    pl.out_sub_stride = (int64_t)n; pl.place = place;
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i], nd = topo[r] / M;
      std::vector<int> grp;
      for (int l = 0; l < M; ++l) grp.push_back(mem[nd * M + l]);
      pccl_comm *g = cached_group(w, grp, 1 + M + nd);
      if (!g) return PCCL_ERR_CUDA;
      pl.rows.push_back({r, g});
    }
    // pull by default (measured faster here); push: staging = work. The direct
    // intra phase is the pull kernel (its push variant has no sub-block layout).
    pl.variant = (!direct && w->p_rs_variant == 1) ? 1 : 0;
    for (int q : mem) {
      pl.send[q] = sendp[q];
      pl.work[q] = work[q];
      pl.recv[q] = work[q];
      pl.out[q] = part[q];
    }
    int s = launch(w, pl, stream);
    if (s) return s;
  } else {
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i];
      if (part_bytes) CK(cudaMemcpyAsync(part[r], sendp[r], part_bytes, cudaMemcpyDeviceToDevice, stream));
    }
  }
  // phase 2: inter reduce-scatter (ring or halving) over the node partials
  if (N > 1) {
    Plan pl;
    pl.coll = PCCL_REDUCE_SCATTER; pl.algo = inter; pl.dtype = dtype; pl.count = n; pl.gs = N;
    if (uniform) pl.force_ctas = chain_ctas;
    if (chain) pl.chain = 2;
    pl.blk = (int64_t)n; pl.istride = (int64_t)n; pl.out_sub_stride = (int64_t)n; pl.place = place;
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int r = ranks[i], j = topo[r] % M;
      std::vector<int> grp;
      for (int nd = 0; nd < N; ++nd) grp.push_back(mem[nd * M + j]);
      pccl_comm *g = cached_group(w, grp, 1 + j);
      if (!g) return PCCL_ERR_CUDA;
      pl.rows.push_back({r, g});
      pl.out[r] = (char *)recvs[i];
    }
    pl.variant = w->p_rs_variant == 1 ? 1 : 0;
    for (int q : mem) {
      pl.send[q] = part[q];
      pl.work[q] = work2[q];
      pl.recv[q] = work2[q];
    }
    return launch(w, pl, stream);
  }
  for (size_t i = 0; i < ranks.size(); ++i) {
    const int r = ranks[i];
    if (n) CK(cudaMemcpyAsync(recvs[i], part[r], n * es, cudaMemcpyDeviceToDevice, stream));
  }
  return PCCL_SUCCESS;
}

}  // namespace

int pccl_ce_available(int device) { return memops(device).ok ? 1 : 0; }

// ---- NVLS multicast segments and collectives --------------------------------
#define CUD(x)                                                                  \
  do {                                                                          \
    const CUresult _r = (x);                                                    \
    if (_r != CUDA_SUCCESS) {                                                   \
      fprintf(stderr, "[pccl_b200] %s failed: CUresult %d\n", #x, (int)_r);     \
      return PCCL_ERR_CUDA;                                                     \
    }                                                                           \
  } while (0)

int pccl_nvls_supported(pccl_world_t w) {
  if (!w || w->emu) return 0;
  DrvNvls &d = drv_nvls();
  if (!d.ok) return 0;
  int v = 0;
  if (d.attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)w->device) != CUDA_SUCCESS) return 0;
  return v ? 1 : 0;
}

static int nvls_slot(pccl_world *w) {
  for (int i = 0; i < 4; ++i)
    if (!w->nvls[i].used) return i;
  return -1;
}

int pccl_nvls_create(pccl_world_t w, size_t bytes, size_t *alloc_bytes, int *fd, int *nvls_id) {
  if (!w || !alloc_bytes || !fd || !nvls_id || bytes == 0) return PCCL_ERR_INVALID_ARGUMENT;
  if (!pccl_nvls_supported(w)) return PCCL_ERR_UNSUPPORTED;
  DrvNvls &d = drv_nvls();
  CK(cudaSetDevice(w->device));
  CK(cudaFree(0));  // the primary context is current
  const int id = nvls_slot(w);
  if (id < 0) return PCCL_ERR_OUT_OF_MEMORY;
  CUmulticastObjectProp mp = nvls_prop(w, bytes);
  size_t gran = 0;
  CUD(d.mcGran(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mc;
  CUD(d.mcCreate(&mc, &mp));
  int h = -1;
  if (d.exportH(&h, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS) {
    d.memRelease(mc);
    return PCCL_ERR_CUDA;
  }
  auto &S = w->nvls[id];
  S = {};
  S.used = true;
  S.mc = mc;
  S.bytes = mp.size;
  S.gran = gran;
  *alloc_bytes = mp.size;
  *fd = h;
  *nvls_id = id;
  return PCCL_SUCCESS;
}

int pccl_nvls_import(pccl_world_t w, int fd, size_t alloc_bytes, int *nvls_id) {
  if (!w || fd < 0 || !alloc_bytes || !nvls_id) return PCCL_ERR_INVALID_ARGUMENT;
  if (!pccl_nvls_supported(w)) return PCCL_ERR_UNSUPPORTED;
  DrvNvls &d = drv_nvls();
  CK(cudaSetDevice(w->device));
  CK(cudaFree(0));
  const int id = nvls_slot(w);
  if (id < 0) return PCCL_ERR_OUT_OF_MEMORY;
  CUmulticastObjectProp mp = nvls_prop(w, alloc_bytes);
  size_t gran = 0;
  CUD(d.mcGran(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle mc;
  CUD(d.importH(&mc, (void *)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  auto &S = w->nvls[id];
  S = {};
  S.used = true;
  S.mc = mc;
  S.bytes = alloc_bytes;
  S.gran = gran;
  *nvls_id = id;
  return PCCL_SUCCESS;
}

// Every rank adds its own device; all must have done so before any binds.
int pccl_nvls_add_device(pccl_world_t w, int id) {
  if (!w || id < 0 || id >= 4 || !w->nvls[id].used) return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  CUD(drv_nvls().mcAddDev((CUmemGenericAllocationHandle)w->nvls[id].mc, (CUdevice)w->device));
  return PCCL_SUCCESS;
}

// Physical memory on my device, bound to the multicast object, mapped twice:
// unicast (my copy, plain loads / stores) and multicast (multimem ops).
int pccl_nvls_bind(pccl_world_t w, int id) {
  if (!w || id < 0 || id >= 4 || !w->nvls[id].used || w->nvls[id].bound) return PCCL_ERR_INVALID_ARGUMENT;
  DrvNvls &d = drv_nvls();
  auto &S = w->nvls[id];
  CK(cudaSetDevice(w->device));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = w->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem;
  CUD(d.memCreate(&mem, S.bytes, &ap, 0));
  S.mem = mem;
  CUD(d.mcBind((CUmemGenericAllocationHandle)S.mc, 0, mem, 0, S.bytes, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = w->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mc = 0;
  CUD(d.reserve(&uc, S.bytes, S.gran, 0, 0));
  CUD(d.map(uc, S.bytes, 0, mem, 0));
  CUD(d.setAccess(uc, S.bytes, &acc, 1));
  CUD(d.reserve(&mc, S.bytes, S.gran, 0, 0));
  CUD(d.map(mc, S.bytes, 0, (CUmemGenericAllocationHandle)S.mc, 0));
  CUD(d.setAccess(mc, S.bytes, &acc, 1));
  S.uc_va = uc;
  S.mc_va = mc;
  S.bound = true;
  CK(cudaMemset((void *)uc, 0, S.bytes));
  CK(cudaDeviceSynchronize());
  return PCCL_SUCCESS;
}

int pccl_nvls_ptr(pccl_world_t w, int id, void **uc, void **mc, size_t *bytes) {
  if (!w || id < 0 || id >= 4 || !w->nvls[id].bound) return PCCL_ERR_INVALID_ARGUMENT;
  if (uc) *uc = (void *)w->nvls[id].uc_va;
  if (mc) *mc = (void *)w->nvls[id].mc_va;
  if (bytes) *bytes = w->nvls[id].bytes;
  return PCCL_SUCCESS;
}

int pccl_nvls_destroy(pccl_world_t w, int id) {
  if (!w || id < 0 || id >= 4 || !w->nvls[id].used) return PCCL_ERR_INVALID_ARGUMENT;
  DrvNvls &d = drv_nvls();
  auto &S = w->nvls[id];
  cudaSetDevice(w->device);
  cudaDeviceSynchronize();
  if (S.mc_va) { d.unmap(S.mc_va, S.bytes); d.addrFree(S.mc_va, S.bytes); }
  if (S.uc_va) { d.unmap(S.uc_va, S.bytes); d.addrFree(S.uc_va, S.bytes); }
  if (S.bound) d.mcUnbind((CUmemGenericAllocationHandle)S.mc, (CUdevice)w->device, 0, S.bytes);
  if (S.mem) d.memRelease((CUmemGenericAllocationHandle)S.mem);
  if (S.mc) d.memRelease((CUmemGenericAllocationHandle)S.mc);
  S = {};
  return PCCL_SUCCESS;
}

// Collectives over a world-spanning communicator (the multicast object spans
// every device of the world). AG: send anywhere on my device, output at
// out_offset of the segment (every rank's copy); RS: input at in_offset of
// the segment (my copy, written before the call), output anywhere.
static int nvls_check(pccl_comm *c, int id, size_t off, size_t bytes_total, const void *p, size_t blk_bytes) {
  pccl_world *w = c ? c->w : nullptr;
  if (!w || w->emu || id < 0 || id >= 4 || !w->nvls[id].bound) return PCCL_ERR_INVALID_ARGUMENT;
  if (c->gs != w->nranks) return PCCL_ERR_UNSUPPORTED;
  if ((off | blk_bytes | (size_t)(uintptr_t)p) & 15) return PCCL_ERR_INVALID_ARGUMENT;
  if (off + bytes_total > w->nvls[id].bytes) return PCCL_ERR_INVALID_ARGUMENT;
  return check_world_err(w);
}

int pccl_nvls_all_gather(pccl_comm_t c, int id, const void *send, size_t out_offset, size_t count, int dtype,
                         void *stream) {
  const size_t es = dt_size(dtype);
  if (!es) return PCCL_ERR_INVALID_ARGUMENT;
  int st = nvls_check(c, id, out_offset, (size_t)(c ? c->gs : 0) * count * es, send, count * es);
  if (st) return st;
  if (count == 0) return PCCL_SUCCESS;
  pccl_world *w = c->w;
  CK(cudaSetDevice(w->device));
  const int me = w->rank;
  Plan pl;
  pl.coll = PCCL_ALL_GATHER;
  pl.algo = A_DIRECT;
  pl.dtype = dtype;
  pl.count = count;
  pl.gs = c->gs;
  pl.blk = pl.istride = pl.send_sub_stride = (int64_t)count;
  pl.variant = 6;
  pl.rows.push_back({me, c});
  pl.send[me] = (char *)send;
  pl.recv[me] = (char *)w->nvls[id].mc_va + out_offset;
  pl.out[me] = (char *)w->nvls[id].uc_va + out_offset;
  // segment and offset enter the call signature: ranks that pass different
  // offsets get LengthMismatch instead of multicasting to different places
  pl.place = (uint32_t)id * 7919u + (uint32_t)(out_offset >> 4) + 1u;
  return launch(w, pl, (cudaStream_t)stream);
}

int pccl_nvls_reduce_scatter(pccl_comm_t c, int id, size_t in_offset, void *recv, size_t recvcount, int dtype,
                             void *stream) {
  if (dtype != PCCL_FLOAT32 && dtype != PCCL_BFLOAT16 && dtype != PCCL_FLOAT16) return PCCL_ERR_UNSUPPORTED;
  const size_t es = dt_size(dtype);
  int st = nvls_check(c, id, in_offset, (size_t)(c ? c->gs : 0) * recvcount * es, recv, recvcount * es);
  if (st) return st;
  if (recvcount == 0) return PCCL_SUCCESS;
  pccl_world *w = c->w;
  CK(cudaSetDevice(w->device));
  const int me = w->rank;
  Plan pl;
  pl.coll = PCCL_REDUCE_SCATTER;
  pl.algo = A_DIRECT;
  pl.dtype = dtype;
  pl.count = recvcount;
  pl.gs = c->gs;
  pl.blk = pl.istride = pl.out_sub_stride = (int64_t)recvcount;
  pl.variant = 6;
  pl.rows.push_back({me, c});
  pl.send[me] = (char *)w->nvls[id].mc_va + in_offset;
  pl.out[me] = (char *)recv;
  pl.place = (uint32_t)id * 7919u + (uint32_t)(in_offset >> 4) + 1u;
  return launch(w, pl, (cudaStream_t)stream);
}
#undef CUD


// ============================================================================
// Point-to-point (transport/base.py:140-152): tagged messages with exact
// (source, tag) FIFO matching, sends that never wait for a matching receive.
// Each (source -> dest) pair owns a ring of PCCL_MBOX_BYTES in the dest's
// flag arena (mapped by every peer). The sender copies a 64-byte frame header
// and the payload into the ring (copy engine, peer memory), then publishes
// its head (bytes written) in the dest's WCTRL word; the receiver drains every
// ring into complete-message buffers in arrival order (so a message waiting
// for its tag never blocks the ring) and publishes its tail (bytes consumed)
// in the sender's WCTRL word. A sender short of ring space drains its own
// incoming rings while it waits, so two ranks exchanging messages larger than
// a ring make progress (sendrecv). Messages larger than a ring travel as
// fragments. Host-driven: this path carries control traffic, never the
// collectives' data.
// ============================================================================
namespace {

constexpr uint64_t kFrameMagic = 0x50434C4C50325000ull;  // "PCLLP2P"
struct Frame {
  uint64_t magic, kind;  // kind 0: message fragment, 1: skip to the ring's end
  int64_t tag;
  uint64_t total, off, len;
  uint64_t pad[2];
};
static_assert(sizeof(Frame) == 64, "frame header is 64 bytes");

char *arena(pccl_world *w, int q) { return w->segs[0].ptr[q]; }
uint64_t *wctrl(pccl_world *w, int q, int idx) {
  return (uint64_t *)arena(w, q) + PCCL_WCTRL_OFF + idx;
}
char *ring(pccl_world *w, int dst, int src) { return arena(w, dst) + PCCL_MBOX_OFF + (size_t)src * PCCL_MBOX_BYTES; }

int p2p_init(pccl_world *w, int me) {
  P2PRank &pr = w->p2p[me];
  if (!pr.stream) CK(cudaStreamCreateWithFlags(&pr.stream, cudaStreamNonBlocking));
  if (!pr.hdr) CK(cudaHostAlloc((void **)&pr.hdr, 64, cudaHostAllocDefault));
  return PCCL_SUCCESS;
}
// Control words and frames move on the rank's own non-blocking stream: a
// mailbox operation never queues behind the collectives on the legacy
// default stream (which may be waiting for the peer that waits for us).
uint64_t read_word(P2PRank &pr, const uint64_t *dev) {
  *(volatile uint64_t *)pr.hdr = 0;
  if (cudaMemcpyAsync(pr.hdr, dev, 8, cudaMemcpyDeviceToHost, pr.stream) != cudaSuccess ||
      cudaStreamSynchronize(pr.stream) != cudaSuccess)
    return 0;
  return *(volatile uint64_t *)pr.hdr;
}
int write_word(P2PRank &pr, uint64_t *dev, uint64_t v) {
  memcpy(pr.hdr, &v, 8);
  CK(cudaMemcpyAsync(dev, pr.hdr, 8, cudaMemcpyHostToDevice, pr.stream));
  CK(cudaStreamSynchronize(pr.stream));
  return PCCL_SUCCESS;
}

// Drain every ring of `me` into complete messages; publish the tails.
int p2p_progress(pccl_world *w, int me) {
  P2PRank &pr = w->p2p[me];
  for (int src = 0; src < w->nranks; ++src) {
    if (src == me) continue;
    const uint64_t head = read_word(pr, wctrl(w, me, PCCL_WCTRL_HEAD + src));
    const uint64_t start = pr.tail_read[src];
    while (pr.tail_read[src] < head) {
      const size_t pos = pr.tail_read[src] % PCCL_MBOX_BYTES;
      Frame f;
      CK(cudaMemcpyAsync(pr.hdr, ring(w, me, src) + pos, sizeof(f), cudaMemcpyDeviceToHost, pr.stream));
      CK(cudaStreamSynchronize(pr.stream));
      memcpy(&f, pr.hdr, sizeof(f));
      if (f.magic != kFrameMagic) return PCCL_ERR_CUDA;  // corrupted ring: never expected
      if (f.kind == 1) {
        pr.tail_read[src] += PCCL_MBOX_BYTES - pos;
        continue;
      }
      P2PMsg &m = pr.partial[src];
      if (!pr.in_partial[src]) {
        m = P2PMsg();
        m.tag = f.tag;
        m.bytes = f.total;
        if (f.total) CK(cudaMallocAsync((void **)&m.dev, f.total, pr.stream));  // stream-ordered: no device-wide sync
        pr.in_partial[src] = true;
      }
      if (f.len) {
        CK(cudaMemcpyAsync(m.dev + f.off, ring(w, me, src) + pos + 64, f.len, cudaMemcpyDeviceToDevice, pr.stream));
        CK(cudaStreamSynchronize(pr.stream));
      }
      m.have += f.len;
      pr.tail_read[src] += 64 + ((f.len + 63) & ~(uint64_t)63);
      if (m.have == m.bytes) {
        pr.unexpected[src].push_back(m);
        pr.in_partial[src] = false;
        m = P2PMsg();
      }
    }
    if (pr.tail_read[src] != start) {
      const int s = write_word(pr, wctrl(w, src, PCCL_WCTRL_TAIL + me), pr.tail_read[src]);
      if (s) return s;
    }
  }
  return PCCL_SUCCESS;
}

int p2p_send(pccl_world *w, int me, int dst, int64_t tag, const void *buf, size_t bytes, bool host) {
  int s = p2p_init(w, me);
  if (s) return s;
  P2PRank &pr = w->p2p[me];
  const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  if (dst == me) {  // self-send: straight into my own queue
    P2PMsg m;
    m.tag = tag;
    m.bytes = m.have = bytes;
    if (bytes) {
      CK(cudaMallocAsync((void **)&m.dev, bytes, pr.stream));
      CK(cudaMemcpyAsync(m.dev, buf, bytes, kind, pr.stream));
      CK(cudaStreamSynchronize(pr.stream));
    }
    pr.unexpected[me].push_back(m);
    return PCCL_SUCCESS;
  }
  const auto t0 = std::chrono::steady_clock::now();
  auto wait_space = [&](uint64_t need) -> int {
    while (true) {
      const uint64_t tail = read_word(pr, wctrl(w, me, PCCL_WCTRL_TAIL + dst));
      if (PCCL_MBOX_BYTES - (pr.head_sent[dst] - tail) >= need) return PCCL_SUCCESS;
      const int e = p2p_progress(w, me);  // keep my own rings draining meanwhile
      if (e) return e;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(w->p_timeout_ms)) return PCCL_ERR_TIMEOUT;
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  };
  const size_t max_frag = PCCL_MBOX_BYTES / 2;
  size_t off = 0;
  do {
    const size_t len = std::min(bytes - off, max_frag);
    const uint64_t need = 64 + ((len + 63) & ~(uint64_t)63);
    size_t pos = pr.head_sent[dst] % PCCL_MBOX_BYTES;
    if (pos + need > PCCL_MBOX_BYTES) {  // frames are contiguous: skip to the ring's start
      const uint64_t rest = PCCL_MBOX_BYTES - pos;
      s = wait_space(rest);
      if (s) return s;
      Frame k{kFrameMagic, 1, 0, 0, 0, 0, {0, 0}};
      memcpy(pr.hdr, &k, 64);
      CK(cudaMemcpyAsync(ring(w, dst, me) + pos, pr.hdr, 64, cudaMemcpyHostToDevice, pr.stream));
      CK(cudaStreamSynchronize(pr.stream));
      pr.head_sent[dst] += rest;
      pos = 0;
    }
    s = wait_space(need);
    if (s) return s;
    Frame f{kFrameMagic, 0, tag, bytes, off, len, {0, 0}};
    memcpy(pr.hdr, &f, 64);
    CK(cudaMemcpyAsync(ring(w, dst, me) + pos, pr.hdr, 64, cudaMemcpyHostToDevice, pr.stream));
    if (len) CK(cudaMemcpyAsync(ring(w, dst, me) + pos + 64, (const char *)buf + off, len, kind, pr.stream));
    CK(cudaStreamSynchronize(pr.stream));  // frame complete in the receiver's memory before the head moves
    pr.head_sent[dst] += need;
    s = write_word(pr, wctrl(w, dst, PCCL_WCTRL_HEAD + me), pr.head_sent[dst]);
    if (s) return s;
    off += len;
  } while (off < bytes);
  return PCCL_SUCCESS;
}

// Blocking receive of the first message from `src` with `tag`. buf == nullptr:
// probe (wait until one is complete, report its size, leave it queued).
int p2p_recv(pccl_world *w, int me, int src, int64_t tag, void *buf, size_t cap, bool host, size_t *bytes) {
  int s = p2p_init(w, me);
  if (s) return s;
  P2PRank &pr = w->p2p[me];
  const auto t0 = std::chrono::steady_clock::now();
  while (true) {
    auto &q = pr.unexpected[src];
    for (auto it = q.begin(); it != q.end(); ++it) {
      if (it->tag != tag) continue;
      if (bytes) *bytes = it->bytes;
      if (!buf) return PCCL_SUCCESS;
      if (cap < it->bytes) return PCCL_ERR_LENGTH_MISMATCH;
      if (it->bytes) {
        CK(cudaMemcpyAsync(buf, it->dev, it->bytes, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                           pr.stream));
        CK(cudaStreamSynchronize(pr.stream));
      }
      if (it->dev) cudaFreeAsync(it->dev, pr.stream);  // cudaFree would synchronise the whole device
      q.erase(it);
      return PCCL_SUCCESS;
    }
    if (src != me) {
      s = p2p_progress(w, me);
      if (s) return s;
      bool got = false;
      for (auto &m : q) got |= m.tag == tag;
      if (got) continue;
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(w->p_timeout_ms)) return PCCL_ERR_TIMEOUT;
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// group ranks -> world ranks; `me` must be this process's rank in real mode
int p2p_ranks(pccl_comm *c, int me, int peer, int *wme, int *wpeer) {
  if (!c || me < 0 || me >= c->gs || peer < 0 || peer >= c->gs) return PCCL_ERR_INDEX_OUT_OF_RANGE;
  if (!c->w->emu && me != c->gi) return PCCL_ERR_INVALID_ARGUMENT;
  *wme = c->members[me];
  *wpeer = c->members[peer];
  CK(cudaSetDevice(c->w->device));
  return check_world_err(c->w);
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char *pccl_error_string(int s) {
  switch (s) {
    case PCCL_SUCCESS: return "success";
    case PCCL_ERR_INVALID_ARGUMENT: return "invalid argument";
    case PCCL_ERR_NON_POWER_OF_TWO: return "algorithm requires a power-of-two group size";
    case PCCL_ERR_NOT_DIVISIBLE: return "buffer not divisible into equal chunks";
    case PCCL_ERR_LENGTH_MISMATCH: return "buffer lengths disagree across ranks";
    case PCCL_ERR_TIMEOUT: return "peer did not arrive before the deadline";
    case PCCL_ERR_PEER_UNREACHABLE: return "peer unreachable";
    case PCCL_ERR_UNSUPPORTED: return "unsupported collective/algorithm/dtype";
    case PCCL_ERR_INVALID_TOPOLOGY: return "invalid topology";
    case PCCL_ERR_INDEX_OUT_OF_RANGE: return "rank out of range";
    case PCCL_ERR_CUDA: return "CUDA runtime error";
    case PCCL_ERR_OUT_OF_MEMORY: return "staging segment too small";
  }
  return "unknown status";
}

int pccl_version(void) { return 100; }

static int world_init(pccl_world *w, int nranks, int rank, int device, bool emu) {
  w->nranks = nranks;
  w->rank = rank;
  w->device = device;
  w->emu = emu;
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  w->sms = prop.multiProcessorCount;
  void *h = nullptr;
  CK(cudaHostAlloc(&h, 64, cudaHostAllocMapped));
  memset(h, 0, 64);
  w->err_host = (volatile int *)h;
  CK(cudaHostGetDevicePointer((void **)&w->err_dev, h, 0));
  if (const char *t = getenv("PCCL_TIMEOUT_MS")) w->p_timeout_ms = atoll(t);
  if (const char *t = getenv("PCCL_CTAS")) w->p_ctas = atoi(t);
  if (const char *t = getenv("PCCL_NSUB")) w->p_nsub = atoi(t);
  if (const char *t = getenv("PCCL_THREADS")) w->p_threads = atoi(t);
  if (const char *t = getenv("PCCL_LOCAL_FENCE")) w->p_local_fence = atoi(t);
  if (const char *t = getenv("PCCL_LL_MAX")) w->p_ll_max = atoll(t);
  if (const char *t = getenv("PCCL_LL128_MAX")) w->p_ll128_max = atoll(t);
  if (const char *t = getenv("PCCL_ITEM_KIB")) w->p_item_kib = atoll(t);
  if (const char *t = getenv("PCCL_PDL")) w->p_pdl = atoi(t);
  if (const char *t = getenv("PCCL_AG_VARIANT")) w->p_ag_variant = atoi(t);  // 5: copy engine (ring / recursive)
  if (const char *t = getenv("PCCL_RS_VARIANT")) w->p_rs_variant = atoi(t);
  if (const char *t = getenv("PCCL_TMA_STAGES")) w->p_tma_stages = atoi(t);
  if (const char *t = getenv("PCCL_TMA_TILE")) w->p_tma_tile = atoi(t);
  int seg = -1;
  int s = pccl_segment_create(w, PCCL_FLAG_BYTES, &seg);
  if (s) return s;
  for (int q = 0; q < nranks; ++q)
    if (w->segs[0].ptr[q]) CK(cudaMemset(w->segs[0].ptr[q], 0, PCCL_FLAG_BYTES));
  CK(cudaDeviceSynchronize());
  return PCCL_SUCCESS;
}

int pccl_world_create(int nranks, int rank, int device, pccl_world_t *out) {
  if (!out || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) return PCCL_ERR_INVALID_ARGUMENT;
  pccl_world *w = new pccl_world();
  int s = world_init(w, nranks, rank, device, false);
  if (s) { delete w; return s; }
  *out = w;
  return PCCL_SUCCESS;
}

int pccl_emu_world_create(int nranks, int device, pccl_world_t *out) {
  if (!out || nranks < 1 || nranks > PCCL_MAXR) return PCCL_ERR_INVALID_ARGUMENT;
  pccl_world *w = new pccl_world();
  int s = world_init(w, nranks, -1, device, true);
  if (s) { delete w; return s; }
  *out = w;
  return PCCL_SUCCESS;
}

int pccl_world_destroy(pccl_world_t w) {
  if (!w) return PCCL_ERR_INVALID_ARGUMENT;
  cudaSetDevice(w->device);
  cudaDeviceSynchronize();
  for (auto &kv : w->comm_cache) delete kv.second;
  for (auto &pr : w->p2p) {
    for (auto &dq : pr.unexpected)
      for (auto &m : dq) cudaFree(m.dev);
    for (auto &m : pr.partial) cudaFree(m.dev);
    if (pr.stream) cudaStreamDestroy(pr.stream);
    if (pr.hdr) cudaFreeHost(pr.hdr);
  }
  for (int i = 0; i < 4; ++i)
    if (w->nvls[i].used) pccl_nvls_destroy(w, i);
  for (int s = kMaxSegs - 1; s >= 0; --s)
    if (w->segs[s].used) pccl_segment_destroy(w, s);
  if (w->err_host) cudaFreeHost((void *)w->err_host);
  if (w->trace_buf) cudaFree(w->trace_buf);
  delete w;
  return PCCL_SUCCESS;
}

int pccl_world_error_detail(pccl_world_t w, int *out16) {
  if (!w || !out16) return PCCL_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < 16; ++i) out16[i] = w->err_host[i];
  return PCCL_SUCCESS;
}

int pccl_world_check(pccl_world_t w) {
  if (!w) return PCCL_ERR_INVALID_ARGUMENT;
  return check_world_err(w);
}

int pccl_world_reset_flags(pccl_world_t w) {
  if (!w) return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  CK(cudaDeviceSynchronize());
  for (int q = 0; q < w->nranks; ++q)
    if (w->segs[0].ptr[q] && w->segs[0].owned[q]) CK(cudaMemset(w->segs[0].ptr[q], 0, PCCL_FLAG_BYTES));
  CK(cudaDeviceSynchronize());
  memset(w->epoch, 0, sizeof(w->epoch));
  memset(w->ce_calls, 0, sizeof(w->ce_calls));
  for (auto &pr : w->p2p) {  // the mailbox counters were cleared with the arena
    for (auto &dq : pr.unexpected) {
      for (auto &m : dq) cudaFree(m.dev);
      dq.clear();
    }
    for (int q = 0; q < PCCL_MAXR; ++q) {
      cudaFree(pr.partial[q].dev);
      pr.partial[q] = P2PMsg();
      pr.in_partial[q] = false;
      pr.head_sent[q] = pr.tail_read[q] = 0;
    }
  }
  for (int i = 0; i < 16; ++i) w->err_host[i] = 0;
  w->poisoned = 0;
  return PCCL_SUCCESS;
}

int pccl_world_set_tuning(pccl_world_t w, int ctas, int nsub, int threads) {
  if (!w || ctas < 0 || ctas > PCCL_MAX_CTAS || nsub < 0 || nsub > 32) return PCCL_ERR_INVALID_ARGUMENT;
  w->p_ctas = ctas;
  if (nsub) w->p_nsub = nsub;
  (void)threads;
  return PCCL_SUCCESS;
}

int pccl_world_set_timeout_ms(pccl_world_t w, int64_t ms) {
  if (!w || ms <= 0) return PCCL_ERR_INVALID_ARGUMENT;
  w->p_timeout_ms = ms;
  return PCCL_SUCCESS;
}

static int64_t *param_ref(pccl_world *w, const char *key) {
  if (!strcmp(key, "ctas")) return &w->p_ctas;
  if (!strcmp(key, "nsub")) return &w->p_nsub;
  if (!strcmp(key, "threads")) return &w->p_threads;
  if (!strcmp(key, "ag_variant")) return &w->p_ag_variant;
  if (!strcmp(key, "rs_variant")) return &w->p_rs_variant;
  if (!strcmp(key, "tma_stages")) return &w->p_tma_stages;
  if (!strcmp(key, "tma_tile")) return &w->p_tma_tile;
  if (!strcmp(key, "timeout_ms")) return &w->p_timeout_ms;
  if (!strcmp(key, "trace")) return &w->p_trace;
  if (!strcmp(key, "local_fence")) return &w->p_local_fence;
  if (!strcmp(key, "staged_bytes")) return &w->p_staged_bytes;
  if (!strcmp(key, "items_per_cta")) return &w->p_items_per_cta;
  if (!strcmp(key, "hier_intra")) return &w->p_hier_intra;
  if (!strcmp(key, "hier_chain")) return &w->p_hier_chain;
  if (!strcmp(key, "pdl")) return &w->p_pdl;
  if (!strcmp(key, "ll_max")) return &w->p_ll_max;
  if (!strcmp(key, "ll128_max")) return &w->p_ll128_max;
  if (!strcmp(key, "item_kib")) return &w->p_item_kib;
  return nullptr;
}

int pccl_world_set_param(pccl_world_t w, const char *key, int64_t value) {
  if (!w || !key) return PCCL_ERR_INVALID_ARGUMENT;
  int64_t *ref = param_ref(w, key);
  const bool is_variant = !strcmp(key, "ag_variant") || !strcmp(key, "rs_variant");
  const bool auto_ok = is_variant || !strcmp(key, "ll_max") || !strcmp(key, "hier_intra");  // -1 = automatic
  if (!ref || value < (auto_ok ? -1 : 0)) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "ctas") && value > PCCL_MAX_CTAS) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "nsub") && (value < 1 || value > 32)) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "threads") && (value < 64 || value > kThreads || value % 32)) return PCCL_ERR_INVALID_ARGUMENT;
  if (is_variant && (value == 6 || value > 8 || (value == 7 && strcmp(key, "rs_variant"))))
    return PCCL_ERR_INVALID_ARGUMENT;  // 4 LL, 5: copy engine (AG) / pipelined push (RS direct), 7: work items
                                       // (RS recursive), 8: LL128 (direct)
  if (!strcmp(key, "items_per_cta") && (value < 1 || value > 16)) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "hier_intra") && value > 1) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "hier_chain") && value > 1) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "tma_stages") && (value < 1 || value > 16)) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "tma_tile") && (value < 16 || value % 16 || value > 200 * 1024)) return PCCL_ERR_INVALID_ARGUMENT;
  if (!strcmp(key, "timeout_ms") && value < 1) return PCCL_ERR_INVALID_ARGUMENT;
  *ref = value;
  return PCCL_SUCCESS;
}

int pccl_world_get_param(pccl_world_t w, const char *key, int64_t *value) {
  if (!w || !key || !value) return PCCL_ERR_INVALID_ARGUMENT;
  int64_t *ref = param_ref(w, key);
  if (!ref) return PCCL_ERR_INVALID_ARGUMENT;
  *value = *ref;
  return PCCL_SUCCESS;
}

int pccl_world_trace_at(pccl_world_t w, int back, uint64_t *host, size_t cap_words, int *rows, int *ctas) {
  if (!w || !host || !rows || !ctas || back < 0) return PCCL_ERR_INVALID_ARGUMENT;
  *rows = w->trace_rows;
  *ctas = w->trace_ctas;
  if (!w->trace_buf || w->trace_seq == 0) return PCCL_SUCCESS;
  const int K = (int)std::max<int64_t>(1, std::min<int64_t>(w->p_trace, PCCL_TRACE_LAUNCHES));
  if (back >= K || back >= w->trace_seq) return PCCL_ERR_INVALID_ARGUMENT;
  const size_t stride = (size_t)PCCL_MAXR * PCCL_MAX_CTAS * PCCL_TRACE_EVENTS;
  const size_t words = (size_t)w->trace_rows * w->trace_ctas * PCCL_TRACE_EVENTS;
  if (cap_words < words) return PCCL_ERR_OUT_OF_MEMORY;
  const int64_t idx = ((w->trace_seq - 1 - back) % K + K) % K;
  CK(cudaSetDevice(w->device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(host, w->trace_buf + stride * (size_t)idx, words * 8, cudaMemcpyDeviceToHost));
  return PCCL_SUCCESS;
}

int pccl_world_trace(pccl_world_t w, uint64_t *host, size_t cap_words, int *rows, int *ctas) {
  return pccl_world_trace_at(w, 0, host, cap_words, rows, ctas);
}

int pccl_segment_create(pccl_world_t w, size_t bytes, int *seg_id) {
  if (!w || !seg_id) return PCCL_ERR_INVALID_ARGUMENT;
  int s = -1;
  for (int i = 0; i < kMaxSegs; ++i)
    if (!w->segs[i].used) { s = i; break; }
  if (s < 0) return PCCL_ERR_OUT_OF_MEMORY;
  CK(cudaSetDevice(w->device));
  Segment &S = w->segs[s];
  S = Segment();
  S.bytes = bytes;
  const size_t alloc = std::max<size_t>(bytes, 256);
  if (w->emu) {
    for (int q = 0; q < w->nranks; ++q) {
      CK(cudaMalloc((void **)&S.ptr[q], alloc));
      S.owned[q] = true;
    }
  } else {
    CK(cudaMalloc((void **)&S.ptr[w->rank], alloc));
    S.owned[w->rank] = true;
  }
  S.used = true;
  w->seg_hi = std::max(w->seg_hi, s + 1);
  *seg_id = s;
  return PCCL_SUCCESS;
}

int pccl_segment_export(pccl_world_t w, int seg_id, void *handle_out) {
  if (!w || w->emu || seg_id < 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used || !handle_out)
    return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, w->segs[seg_id].ptr[w->rank]));
  memcpy(handle_out, &h, sizeof(h));
  return PCCL_SUCCESS;
}

int pccl_segment_import(pccl_world_t w, int seg_id, const void *handles) {
  if (!w || w->emu || seg_id < 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used || !handles)
    return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  Segment &S = w->segs[seg_id];
  for (int q = 0; q < w->nranks; ++q) {
    if (q == w->rank || S.ptr[q]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char *)handles + (size_t)q * PCCL_IPC_HANDLE_BYTES, sizeof(h));
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      fprintf(stderr, "[pccl_b200] rank %d cannot map segment %d of rank %d: %s\n", w->rank, seg_id, q,
              cudaGetErrorString(e));
      return PCCL_ERR_PEER_UNREACHABLE;
    }
    S.ptr[q] = (char *)p;
    S.opened[q] = true;
  }
  return PCCL_SUCCESS;
}

// ---- registration of caller-owned memory (e.g. torch caching-allocator
// tensors): the peers map the allocation that contains the buffer (CUDA IPC
// handle of the allocation base + offset), so collectives read / write the
// registered buffers zero-copy, exactly like World segments.
static int alloc_seg(pccl_world *w) {
  for (int i = 1; i < kMaxSegs; ++i)
    if (!w->segs[i].used) return i;
  return -1;
}

int pccl_segment_register(pccl_world_t w, void *ptr, size_t bytes, int *seg_id) {
  if (!w || w->emu || !ptr || !seg_id) return PCCL_ERR_INVALID_ARGUMENT;
  const int s = alloc_seg(w);
  if (s < 0) return PCCL_ERR_OUT_OF_MEMORY;
  Segment &S = w->segs[s];
  S = Segment();
  S.bytes = bytes;
  S.reg = true;
  S.ptr[w->rank] = (char *)ptr;
  S.used = true;
  w->seg_hi = std::max(w->seg_hi, s + 1);
  *seg_id = s;
  return PCCL_SUCCESS;
}

int pccl_emu_segment_register(pccl_world_t w, void *const *ptrs, size_t bytes, int *seg_id) {
  if (!w || !w->emu || !ptrs || !seg_id) return PCCL_ERR_INVALID_ARGUMENT;
  const int s = alloc_seg(w);
  if (s < 0) return PCCL_ERR_OUT_OF_MEMORY;
  Segment &S = w->segs[s];
  S = Segment();
  S.bytes = bytes;
  S.reg = true;
  for (int q = 0; q < w->nranks; ++q) {
    if (!ptrs[q]) return PCCL_ERR_INVALID_ARGUMENT;
    S.ptr[q] = (char *)ptrs[q];
  }
  S.used = true;
  w->seg_hi = std::max(w->seg_hi, s + 1);
  *seg_id = s;
  return PCCL_SUCCESS;
}

using MemGetAddressRangeFn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
static MemGetAddressRangeFn mem_range_fn() {
  static MemGetAddressRangeFn f = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = (MemGetAddressRangeFn)fp;
    else
      cudaGetLastError();
  });
  return f;
}

int pccl_segment_register_export(pccl_world_t w, int seg_id, void *handle_out) {
  if (!w || w->emu || seg_id <= 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used || !w->segs[seg_id].reg ||
      !handle_out)
    return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  MemGetAddressRangeFn range = mem_range_fn();
  if (!range) return PCCL_ERR_UNSUPPORTED;
  CUdeviceptr base = 0;
  size_t size = 0;
  char *p = w->segs[seg_id].ptr[w->rank];
  if (range(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) return PCCL_ERR_INVALID_ARGUMENT;  // not device memory
  if ((char *)base + size < p + w->segs[seg_id].bytes) return PCCL_ERR_INVALID_ARGUMENT;     // spans allocations
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void *)base) != cudaSuccess) {  // e.g. VMM / expandable-segment memory
    cudaGetLastError();
    return PCCL_ERR_UNSUPPORTED;
  }
  const uint64_t off = (uint64_t)(p - (char *)base), sz = (uint64_t)size;
  memcpy(handle_out, &h, sizeof(h));
  memcpy((char *)handle_out + PCCL_IPC_HANDLE_BYTES, &off, 8);
  memcpy((char *)handle_out + PCCL_IPC_HANDLE_BYTES + 8, &sz, 8);
  return PCCL_SUCCESS;
}

int pccl_segment_register_import(pccl_world_t w, int seg_id, const void *handles) {
  if (!w || w->emu || seg_id <= 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used || !w->segs[seg_id].reg ||
      !handles)
    return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  Segment &S = w->segs[seg_id];
  for (int q = 0; q < w->nranks; ++q) {
    if (q == w->rank || S.ptr[q]) continue;
    const char *hq = (const char *)handles + (size_t)q * PCCL_REG_HANDLE_BYTES;
    uint64_t off = 0;
    memcpy(&off, hq + PCCL_IPC_HANDLE_BYTES, 8);
    std::string key((const char *)&q, sizeof(q));
    key.append(hq, PCCL_IPC_HANDLE_BYTES);
    auto it = w->ipc_open.find(key);
    char *base = nullptr;
    if (it != w->ipc_open.end()) {
      base = it->second.first;
      it->second.second++;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, hq, sizeof(h));
      void *b = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        fprintf(stderr, "[pccl_b200] rank %d cannot map registered buffer of rank %d: %s\n", w->rank, q,
                cudaGetErrorString(e));
        return PCCL_ERR_PEER_UNREACHABLE;
      }
      base = (char *)b;
      w->ipc_open[key] = {base, 1};
    }
    S.ipc_base[q] = base;
    S.ptr[q] = base + off;
  }
  return PCCL_SUCCESS;
}

int pccl_segment_ptr(pccl_world_t w, int seg_id, int rank, void **ptr, size_t *bytes) {
  if (!w || seg_id < 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used || rank < 0 || rank >= w->nranks)
    return PCCL_ERR_INVALID_ARGUMENT;
  if (ptr) *ptr = w->segs[seg_id].ptr[rank];
  if (bytes) *bytes = w->segs[seg_id].bytes;
  return PCCL_SUCCESS;
}

int pccl_segment_destroy(pccl_world_t w, int seg_id) {
  if (!w || seg_id < 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used) return PCCL_ERR_INVALID_ARGUMENT;
  cudaSetDevice(w->device);
  cudaDeviceSynchronize();
  Segment &S = w->segs[seg_id];
  for (int q = 0; q < w->nranks; ++q) {
    if (S.opened[q]) cudaIpcCloseMemHandle(S.ptr[q]);
    if (S.owned[q]) cudaFree(S.ptr[q]);
    if (S.ipc_base[q]) {  // registered: drop this segment's reference on the peer allocation's mapping
      for (auto it = w->ipc_open.begin(); it != w->ipc_open.end(); ++it)
        if (it->second.first == S.ipc_base[q]) {
          if (--it->second.second == 0) {
            cudaIpcCloseMemHandle(it->second.first);
            w->ipc_open.erase(it);
          }
          break;
        }
    }
  }
  S = Segment();
  if (w->staging == seg_id) w->staging = -1;
  return PCCL_SUCCESS;
}

int pccl_world_set_staging(pccl_world_t w, int seg_id) {
  if (!w || seg_id <= 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used) return PCCL_ERR_INVALID_ARGUMENT;
  w->staging = seg_id;
  return PCCL_SUCCESS;
}

size_t pccl_staging_bytes(int collective, int algo, int gs, size_t count, int dtype) {
  // Mirrors the Binder layouts of do_all_gather / do_reduce_scatter /
  // do_hier_*; algo 3 = hierarchical. count = AG block / RS chunk elements.
  const size_t es = dt_size(dtype);
  if (gs < 1) gs = 1;
  const size_t full = align256((size_t)gs * count * es), blk = align256(count * es);
  if (collective == PCCL_ALL_GATHER) return full + blk;
  if (algo == 3) return 4 * full;
  return algo == A_DIRECT ? full + blk : 2 * full;  // direct LL may bounce a misaligned input and output
}

int pccl_comm_create(pccl_world_t w, const int *members, int n, int comm_id, pccl_comm_t *out) {
  if (!w || !members || !out || n < 1 || n > w->nranks) return PCCL_ERR_INVALID_ARGUMENT;
  pccl_comm *c = new pccl_comm();
  c->w = w;
  c->gs = n;
  c->comm_id = comm_id;
  for (int i = 0; i < n; ++i) {
    if (members[i] < 0 || members[i] >= w->nranks || (c->mask >> members[i]) & 1u) {
      delete c;
      return PCCL_ERR_INVALID_ARGUMENT;
    }
    c->members[i] = members[i];
    c->mask |= 1u << members[i];
    if (!w->emu && members[i] == w->rank) c->gi = i;
  }
  if (!w->emu && c->gi < 0) {
    delete c;
    return PCCL_ERR_INDEX_OUT_OF_RANGE;
  }
  c->slot = slot_for(w, c->mask);
  if (c->slot < 0) {
    delete c;
    return PCCL_ERR_OUT_OF_MEMORY;
  }
  *out = c;
  return PCCL_SUCCESS;
}

int pccl_comm_epoch(pccl_comm_t c, int member, uint64_t *epoch) {
  if (!c || !epoch || member < 0 || member >= c->gs) return PCCL_ERR_INVALID_ARGUMENT;
  pccl_world *w = c->w;
  const int r = c->members[member];
  if (!w->emu && r != w->rank) return PCCL_ERR_INVALID_ARGUMENT;
  CK(cudaSetDevice(w->device));
  CK(cudaDeviceSynchronize());
  const uint64_t *ctrl = (const uint64_t *)w->segs[0].ptr[r] + (size_t)c->slot * PCCL_SLOT_WORDS + PCCL_CTRL_OFF;
  CK(cudaMemcpy(epoch, ctrl, 8, cudaMemcpyDeviceToHost));
  return PCCL_SUCCESS;
}

int pccl_comm_destroy(pccl_comm_t c) {
  if (!c) return PCCL_ERR_INVALID_ARGUMENT;
  delete c;
  return PCCL_SUCCESS;
}

int pccl_comm_size(pccl_comm_t c, int *size) {
  if (!c || !size) return PCCL_ERR_INVALID_ARGUMENT;
  *size = c->gs;
  return PCCL_SUCCESS;
}

int pccl_comm_rank(pccl_comm_t c, int *rank) {
  if (!c || !rank) return PCCL_ERR_INVALID_ARGUMENT;
  *rank = c->gi;
  return PCCL_SUCCESS;
}

int pccl_send(pccl_comm_t c, int me, int dst, int64_t tag, const void *buf, size_t bytes, int host) {
  int wme, wdst;
  int s = p2p_ranks(c, me, dst, &wme, &wdst);
  if (s) return s;
  if (bytes && !buf) return PCCL_ERR_INVALID_ARGUMENT;
  return p2p_send(c->w, wme, wdst, tag, buf, bytes, host != 0);
}

int pccl_recv(pccl_comm_t c, int me, int src, int64_t tag, void *buf, size_t cap, int host, size_t *bytes) {
  int wme, wsrc;
  int s = p2p_ranks(c, me, src, &wme, &wsrc);
  if (s) return s;
  return p2p_recv(c->w, wme, wsrc, tag, buf, cap, host != 0, bytes);
}

int pccl_all_gather(pccl_comm_t c, int algo, const void *send, void *recv, size_t count, int dtype, void *stream) {
  if (!c || c->w->emu) return PCCL_ERR_INVALID_ARGUMENT;
  int e = check_world_err(c->w);
  if (e) return e;
  const void *s[1] = {send};
  void *r[1] = {recv};
  return do_all_gather(c, algo, one(c->w->rank), s, r, count, dtype, (cudaStream_t)stream);
}

int pccl_reduce_scatter(pccl_comm_t c, int algo, int order, const void *send, void *recv, size_t recvcount, int dtype,
                        void *stream) {
  if (!c || c->w->emu) return PCCL_ERR_INVALID_ARGUMENT;
  int e = check_world_err(c->w);
  if (e) return e;
  const void *s[1] = {send};
  void *r[1] = {recv};
  return do_reduce_scatter(c, algo, order, one(c->w->rank), s, r, recvcount, dtype, (cudaStream_t)stream);
}

int pccl_hier_all_gather(pccl_world_t w, int N, int M, int inter, const void *send, void *recv, size_t count, int dtype,
                         void *stream) {
  if (!w || w->emu) return PCCL_ERR_INVALID_ARGUMENT;
  int e = check_world_err(w);
  if (e) return e;
  const void *s[1] = {send};
  void *r[1] = {recv};
  return do_hier_all_gather(w, iota_ranks(w->nranks), N, M, inter, one(w->rank), s, r, count, dtype,
                            (cudaStream_t)stream);
}

int pccl_hier_reduce_scatter(pccl_world_t w, int N, int M, int inter, const void *send, void *recv, size_t recvcount,
                             int dtype, void *stream) {
  if (!w || w->emu) return PCCL_ERR_INVALID_ARGUMENT;
  int e = check_world_err(w);
  if (e) return e;
  const void *s[1] = {send};
  void *r[1] = {recv};
  return do_hier_reduce_scatter(w, iota_ranks(w->nranks), N, M, inter, one(w->rank), s, r, recvcount, dtype,
                                (cudaStream_t)stream);
}

int pccl_emu_all_gather(pccl_comm_t c, int algo, const void *const *sends, void *const *recvs, size_t count, int dtype,
                        void *stream) {
  if (!c || !c->w->emu || !sends || !recvs) return PCCL_ERR_INVALID_ARGUMENT;
  std::vector<int> ranks(c->members, c->members + c->gs);
  return do_all_gather(c, algo, ranks, sends, recvs, count, dtype, (cudaStream_t)stream);
}

int pccl_emu_reduce_scatter(pccl_comm_t c, int algo, int order, const void *const *sends, void *const *recvs,
                            size_t recvcount, int dtype, void *stream) {
  if (!c || !c->w->emu || !sends || !recvs) return PCCL_ERR_INVALID_ARGUMENT;
  std::vector<int> ranks(c->members, c->members + c->gs);
  return do_reduce_scatter(c, algo, order, ranks, sends, recvs, recvcount, dtype, (cudaStream_t)stream);
}

int pccl_emu_hier_all_gather(pccl_world_t w, int N, int M, int inter, const void *const *sends, void *const *recvs,
                             size_t count, int dtype, void *stream) {
  if (!w || !w->emu || !sends || !recvs) return PCCL_ERR_INVALID_ARGUMENT;
  std::vector<int> ranks;
  for (int r = 0; r < w->nranks; ++r) ranks.push_back(r);
  return do_hier_all_gather(w, ranks, N, M, inter, ranks, sends, recvs, count, dtype, (cudaStream_t)stream);
}

int pccl_emu_hier_reduce_scatter(pccl_world_t w, int N, int M, int inter, const void *const *sends, void *const *recvs,
                                 size_t recvcount, int dtype, void *stream) {
  if (!w || !w->emu || !sends || !recvs) return PCCL_ERR_INVALID_ARGUMENT;
  std::vector<int> ranks;
  for (int r = 0; r < w->nranks; ++r) ranks.push_back(r);
  return do_hier_reduce_scatter(w, ranks, N, M, inter, ranks, sends, recvs, recvcount, dtype, (cudaStream_t)stream);
}

// Over any communicator of N*M members (hierarchy.py:129-134 only requires
// the communicator size to match the topology): topology rank g is member g.
int pccl_hier_all_gather_comm(pccl_comm_t c, int N, int M, int inter, const void *send, void *recv, size_t count,
                              int dtype, void *stream) {
  if (!c || c->w->emu) return PCCL_ERR_INVALID_ARGUMENT;
  int e = check_world_err(c->w);
  if (e) return e;
  const void *s[1] = {send};
  void *r[1] = {recv};
  return do_hier_all_gather(c->w, std::vector<int>(c->members, c->members + c->gs), N, M, inter, one(c->w->rank), s, r,
                            count, dtype, (cudaStream_t)stream);
}

int pccl_hier_reduce_scatter_comm(pccl_comm_t c, int N, int M, int inter, const void *send, void *recv,
                                  size_t recvcount, int dtype, void *stream) {
  if (!c || c->w->emu) return PCCL_ERR_INVALID_ARGUMENT;
  int e = check_world_err(c->w);
  if (e) return e;
  const void *s[1] = {send};
  void *r[1] = {recv};
  return do_hier_reduce_scatter(c->w, std::vector<int>(c->members, c->members + c->gs), N, M, inter, one(c->w->rank),
                                s, r, recvcount, dtype, (cudaStream_t)stream);
}

int pccl_emu_hier_all_gather_comm(pccl_comm_t c, int N, int M, int inter, const void *const *sends,
                                  void *const *recvs, size_t count, int dtype, void *stream) {
  if (!c || !c->w->emu || !sends || !recvs) return PCCL_ERR_INVALID_ARGUMENT;
  std::vector<int> mem(c->members, c->members + c->gs);
  return do_hier_all_gather(c->w, mem, N, M, inter, mem, sends, recvs, count, dtype, (cudaStream_t)stream);
}

int pccl_emu_hier_reduce_scatter_comm(pccl_comm_t c, int N, int M, int inter, const void *const *sends,
                                      void *const *recvs, size_t recvcount, int dtype, void *stream) {
  if (!c || !c->w->emu || !sends || !recvs) return PCCL_ERR_INVALID_ARGUMENT;
  std::vector<int> mem(c->members, c->members + c->gs);
  return do_hier_reduce_scatter(c->w, mem, N, M, inter, mem, sends, recvs, recvcount, dtype, (cudaStream_t)stream);
}

int pccl_emu_debug_meta_skew(pccl_world_t w, int rank, uint32_t xor_mask) {
  if (!w || rank < 0 || rank >= w->nranks) return PCCL_ERR_INVALID_ARGUMENT;
  w->meta_skew[rank] = xor_mask & 0x7fffffff;
  return PCCL_SUCCESS;
}

int pccl_probe(pccl_world_t w, int seg_id, int mode, uint32_t dst_mask, size_t bytes, int ctas, void *stream) {
  if (!w || w->emu || seg_id <= 0 || seg_id >= kMaxSegs || !w->segs[seg_id].used || bytes % 16 || ctas < 1) return PCCL_ERR_INVALID_ARGUMENT;
  const Segment &S = w->segs[seg_id];
  if (2 * bytes > S.bytes) return PCCL_ERR_INVALID_ARGUMENT;
  LaunchParams P;
  memset(&P, 0, sizeof(P));
  // peers' second half is the remote target; my first half is the local side
  for (int q = 0; q < w->nranks; ++q) P.recv[q] = S.ptr[q] ? S.ptr[q] + S.bytes / 2 : nullptr;
  dst_mask &= ~(1u << w->rank);
  CK(cudaSetDevice(w->device));
  if (mode == 4 || mode == 5) {
    P.tma_stages = (int)w->p_tma_stages;
    P.tma_tile = (uint32_t)w->p_tma_tile;
    const size_t smem = (size_t)P.tma_stages * P.tma_tile + 8 * (size_t)P.tma_stages;
    CK(cudaFuncSetAttribute((const void *)k_probe_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_probe_tma<<<ctas, kThreads, smem, (cudaStream_t)stream>>>(S.ptr[w->rank], P, dst_mask, (int64_t)(bytes / 16), mode);
  } else {
    k_probe<<<ctas, kThreads, 0, (cudaStream_t)stream>>>(S.ptr[w->rank], P, dst_mask, (int64_t)(bytes / 16), mode);
  }
  CK(cudaGetLastError());
  return PCCL_SUCCESS;
}

int pccl_shuffle(int direction, const void *in, void *out, int N, int M, size_t block_len, int dtype, void *stream) {
  const size_t es = dt_size(dtype);
  if (!es || N < 1 || M < 1 || (direction != 0 && direction != 1)) return PCCL_ERR_INVALID_ARGUMENT;
  const size_t total = (size_t)N * M * block_len * es;
  if (total == 0) return PCCL_SUCCESS;
  // direction 0 (local-major -> global): input is an M x N grid -> out N x M
  const int A = direction == 0 ? N : M;  // output-major dimension
  const int Bd = direction == 0 ? M : N;
  uint64_t acc = (uint64_t)(uintptr_t)in | (uint64_t)(uintptr_t)out | (uint64_t)(block_len * es);
  int U = 16;
  while (U > 1 && (acc & (uint64_t)(U - 1))) U >>= 1;
  const int64_t blk = (int64_t)(block_len * es / U);
  const int64_t units = (int64_t)A * Bd * blk;
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((units + kThreads - 1) / kThreads, (int64_t)sms * 4);
  cudaStream_t s = (cudaStream_t)stream;
  switch (U) {
    case 16: k_shuffle<16><<<grid, kThreads, 0, s>>>((const char *)in, (char *)out, A, Bd, blk); break;
    case 8: k_shuffle<8><<<grid, kThreads, 0, s>>>((const char *)in, (char *)out, A, Bd, blk); break;
    case 4: k_shuffle<4><<<grid, kThreads, 0, s>>>((const char *)in, (char *)out, A, Bd, blk); break;
    case 2: k_shuffle<2><<<grid, kThreads, 0, s>>>((const char *)in, (char *)out, A, Bd, blk); break;
    default: k_shuffle<1><<<grid, kThreads, 0, s>>>((const char *)in, (char *)out, A, Bd, blk); break;
  }
  CK(cudaGetLastError());
  return PCCL_SUCCESS;
}

int pccl_copy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height, void *stream) {
  if (width == 0 || height == 0) return PCCL_SUCCESS;
  if (!dst || !src || dpitch < width || spitch < width) return PCCL_ERR_INVALID_ARGUMENT;
  if (cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, (cudaStream_t)stream) != cudaSuccess) {
    cudaGetLastError();
    return PCCL_ERR_CUDA;
  }
  return PCCL_SUCCESS;
}

int pccl_reduce_inplace(void *acc, const void *other, size_t count, int dtype, void *stream) {
  if (count == 0) return PCCL_SUCCESS;
  if (!acc || !other) return PCCL_ERR_INVALID_ARGUMENT;
  const size_t es = dt_size(dtype);
  const bool vec = (((uintptr_t)acc | (uintptr_t)other | (count * es)) & 15) == 0;
  const int64_t n = vec ? (int64_t)(count * es / 16) : (int64_t)count;
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, (int64_t)sms * 4);
  cudaStream_t s = (cudaStream_t)stream;
#define RI(DT)                                                                                      \
  if (vec) k_reduce_inplace<DT, true><<<grid, kThreads, 0, s>>>((char *)acc, (const char *)other, n); \
  else k_reduce_inplace<DT, false><<<grid, kThreads, 0, s>>>((char *)acc, (const char *)other, n);
  switch (dtype) {
    case PCCL_FLOAT32: RI(DT_F32); break;
    case PCCL_BFLOAT16: RI(DT_BF16); break;
    case PCCL_FLOAT16: RI(DT_F16); break;
    default: return PCCL_ERR_UNSUPPORTED;
  }
#undef RI
  CK(cudaGetLastError());
  return PCCL_SUCCESS;
}

// ---------------------------------------------------------------------------
// schedule introspection: rows (step, src, dst, nbytes) — dst pulls from src
// ---------------------------------------------------------------------------
namespace {
struct Rows {
  int64_t *rows;
  int cap, n = 0, step = 0;
  bool overflow = false;
  void add(int src, int dst, int64_t bytes) {
    if (n >= cap) { overflow = true; return; }
    int64_t *r = rows + 4 * n++;
    r[0] = step; r[1] = src; r[2] = dst; r[3] = bytes;
  }
};

// Emits the steps of one flat collective over `members` (concurrent groups
// are merged by the caller by resetting `step` to the phase's start).
int flat_steps(Rows &R, int coll, int algo, const std::vector<int> &mem, int64_t m_bytes, int step0) {
  const int gs = (int)mem.size();
  if (m_bytes % gs) return PCCL_ERR_NOT_DIVISIBLE;
  const int64_t blk = m_bytes / gs;
  if (gs == 1) return PCCL_SUCCESS;
  if (algo == A_RING) {
    for (int s = 0; s < gs - 1; ++s) {
      R.step = step0 + s;
      for (int gi = 0; gi < gs; ++gi) R.add(mem[ring_prev(gi, gs)], mem[gi], blk);
    }
  } else if (algo == A_REC) {
    if (!is_pow2(gs)) return PCCL_ERR_NON_POWER_OF_TWO;
    int L = 0;
    while ((1 << L) < gs) ++L;
    for (int k = 0; k < L; ++k) {
      R.step = step0 + k;
      for (int gi = 0; gi < gs; ++gi) {
        if (coll == PCCL_ALL_GATHER) R.add(mem[recdbl_partner(gi, k)], mem[gi], (int64_t)(1 << k) * blk);
        else R.add(mem[rechalf_partner(gi, gs, k)], mem[gi], (int64_t)(gs >> (k + 1)) * blk);
      }
    }
  } else if (algo == A_DIRECT) {
    R.step = step0;
    for (int gi = 0; gi < gs; ++gi)
      for (int q = 0; q < gs; ++q)
        if (q != gi) R.add(mem[q], mem[gi], blk);
  } else {
    return PCCL_ERR_INVALID_ARGUMENT;
  }
  return PCCL_SUCCESS;
}

int nsteps(int algo, int gs) {
  if (gs == 1) return 0;
  if (algo == A_RING) return gs - 1;
  if (algo == A_DIRECT) return 1;
  int L = 0;
  while ((1 << L) < gs) ++L;
  return L;
}
}  // namespace

int pccl_schedule(int coll, int algo, int inter, int N, int M, size_t m_bytes, int64_t *rows, int cap, int *nrows) {
  if (!rows || !nrows || N < 1 || M < 1 || N * M > PCCL_MAXR) return PCCL_ERR_INVALID_ARGUMENT;
  Rows R{rows, cap};
  const int p = N * M;
  int s = PCCL_SUCCESS;
  if (algo != 3) {  // flat over the world
    std::vector<int> mem;
    for (int g = 0; g < p; ++g) mem.push_back(g);
    s = flat_steps(R, coll, algo, mem, (int64_t)m_bytes, 0);
  } else {  // hierarchical: inter phase (groups j) and intra phase (groups n)
    if ((int64_t)m_bytes % p) return PCCL_ERR_NOT_DIVISIBLE;
    if (inter == A_REC && !is_pow2(N)) return PCCL_ERR_NON_POWER_OF_TWO;
    auto inter_phase = [&](int step0) {
      for (int j = 0; j < M && !s; ++j) {
        std::vector<int> mem;
        for (int n = 0; n < N; ++n) mem.push_back(n * M + j);
        s = flat_steps(R, coll, inter, mem, (int64_t)m_bytes / M, step0);
      }
      return step0 + nsteps(inter, N);
    };
    auto intra_phase = [&](int step0) {
      for (int n = 0; n < N && !s; ++n) {
        std::vector<int> mem;
        for (int l = 0; l < M; ++l) mem.push_back(n * M + l);
        s = flat_steps(R, coll, A_RING, mem, (int64_t)m_bytes, step0);
      }
      return step0 + nsteps(A_RING, M);
    };
    if (coll == PCCL_ALL_GATHER) intra_phase(inter_phase(0));
    else inter_phase(intra_phase(0));
  }
  *nrows = R.n;
  if (s) return s;
  return R.overflow ? PCCL_ERR_OUT_OF_MEMORY : PCCL_SUCCESS;
}

}  // extern "C"
