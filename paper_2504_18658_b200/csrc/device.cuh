// device.cuh — launch parameters, cross-GPU flag protocol and data-path
// primitives shared by every collective kernel (sm_100a).
//
// Protocol (replaces the tagged P2P transport, collkit/transport/base.py:3-20):
//   * every rank owns a flag arena (segment 0) mapped into every peer;
//   * a group (communicator) owns one flag *slot* in every member's arena;
//   * the WRITER of a signal stores into the READER's arena, the reader polls
//     its own memory (ld.acquire.sys), the writer publishes with st.release.sys
//     after a CTA barrier — one NVLink write per signal, no remote polling;
//   * READY[src][cta] carries a monotonic progress counter
//     (epoch << 32 | hash << 10 | units_done) so flags are never reset: the
//     per-group epoch plays the role of next_base_tag()'s sequence number
//     (transport/base.py:131-138);
//   * DONE[src][cta] = epoch once src has finished reading this rank's buffers
//     (the WAR guard that lets the caller reuse them after the call);
//   * the READY word also carries 22 bits of the call-signature hash
//     (count, dtype, algorithm, variant, placement), checked on every wait: a
//     cross-rank mismatch raises LengthMismatch like from_payload
//     (collectives.py:36-42);
//   * a wait that sees ABORT_BIT, or exceeds the %globaltimer deadline, records
//     the error in the world's host-mapped error word and floods ABORT into
//     every member's slot so no CTA on any GPU is left spinning.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#ifndef PCCL_MAXR
#define PCCL_MAXR 16
#endif
#define PCCL_MAX_CTAS 320
#define PCCL_NSLOTS 256
#define PCCL_CTRL_OFF (4 * PCCL_MAXR * PCCL_MAX_CTAS)
#define PCCL_SLOT_WORDS (PCCL_CTRL_OFF + 64)  // + CTRL: [0] last completed epoch, [1] CTA exit counter,
                                              //   [2] work-item counter (direct kernels, see for_items),
                                              //   [3..10] per-step item counters (k_rs_rec_items),
                                              //   [11] CTAs done with the final unit (cta_signal_rank)
#define PCCL_SLOT_BYTES (PCCL_SLOT_WORDS * 8)
// After the slots: world-level control words, then the LL (low-latency)
// message regions (see "LL protocol" below). Both live in segment 0, so every
// peer already has them mapped.
#define PCCL_WCTRL_OFF ((size_t)PCCL_NSLOTS * PCCL_SLOT_WORDS)  // words: [q] LL messages exchanged with world rank q
#define PCCL_WCTRL_WORDS 128
#define PCCL_LL_OFF (PCCL_WCTRL_OFF + PCCL_WCTRL_WORDS)  // words
#define PCCL_LL_HDR_BYTES 256
#define PCCL_LL_MAX_PAYLOAD ((size_t)1 << 20)  // payload bytes per (src -> dst) message
#define PCCL_LL_REGION_BYTES (PCCL_LL_HDR_BYTES + 2 * PCCL_LL_MAX_PAYLOAD)
// After the LL regions: the point-to-point mailboxes (host-driven send / recv,
// see "point-to-point" in pccl_b200.cu): per source rank one ring of
// PCCL_MBOX_BYTES in the receiver's arena. WCTRL words [16 + s]: bytes rank s
// has written into my ring (its head); [32 + d]: bytes rank d has consumed of
// my messages (my tail at d).
#define PCCL_MBOX_OFF ((PCCL_LL_OFF * 8 + (size_t)2 * PCCL_MAXR * PCCL_LL_REGION_BYTES + 4095) & ~(size_t)4095)  // bytes
#define PCCL_MBOX_BYTES ((size_t)2 << 20)
#define PCCL_WCTRL_HEAD 16
#define PCCL_WCTRL_TAIL 32
// WCTRL [48]: device-side mirror of the world error word. Spinning CTAs poll
// it instead of the host-mapped error word: 128 CTAs reading host memory at
// once stalled a kernel's exits by up to 120 us (profiles/r2_overhead_p4.md).
#define PCCL_WCTRL_ERR 48
// After the mailboxes: the LL128 message regions (line protocol for mid-size
// direct all-gathers, "LL128" below). Separate from the LL regions so that a
// receiver of one format never polls stale payload of the other; its channel
// counters are WCTRL [64 + q].
#define PCCL_WCTRL_LL128 64
#define PCCL_LL128_LINES 16384  // 128-byte lines per message (2 MiB)
#define PCCL_LL128_MAX_PAYLOAD ((size_t)PCCL_LL128_LINES * 120)
#define PCCL_LL128_REGION_BYTES (PCCL_LL_HDR_BYTES + (size_t)PCCL_LL128_LINES * 128)
#define PCCL_LL128_OFF (PCCL_MBOX_OFF + (size_t)PCCL_MAXR * PCCL_MBOX_BYTES)  // bytes
#define PCCL_FLAG_BYTES (PCCL_LL128_OFF + (size_t)2 * PCCL_MAXR * PCCL_LL128_REGION_BYTES)
#define PCCL_ABORT_BIT (1ull << 63)

namespace pccl {

enum FlagKind { F_READY = 0, F_DONE = 1, F_META = 2, F_ITEM = 3 };  // F_ITEM: per-item progress (item kernels)
enum Dt { DT_F32 = 0, DT_BF16 = 1, DT_F16 = 2 };
enum Algo { A_DIRECT = 0, A_RING = 1, A_REC = 2 };
enum Order { O_RING = 0, O_REC = 1, O_RANK = 2 };

// One launch = one or more groups of equal size `gs`; launch row y (blockIdx.y)
// acts for world rank row_rank[y]. Real mode has a single row; emulation mode
// has one row per emulated rank. Layout fields are in *units* (a unit is a
// 16-byte vector when the path is vectorised, else one element / U bytes).
struct LaunchParams {
  int gs;           // group size
  int ctas;         // CTAs per row (== gridDim.x)
  int nsub;         // pipeline sub-slices per CTA slice
  int nsubblk;      // sub-blocks per member block / chunk (hierarchical layouts)
  int local_copy;   // AG: copy own send block into recv
  int order;        // direct RS fold order
  int skip_exit;    // 1: no DONE barrier (buffers not reused while peers read)
  int variant;      // data-movement variant (experiments / tuning)
  int tma_stages;   // TMA ring depth
  uint32_t tma_tile;  // TMA tile bytes
  int local_fence;  // 1: pull-kernel signals fence at gpu scope (data is in the writer's own HBM)
  int wire;         // direct RS fold: round the partial to the storage type after every add (= step-wise algorithms)
  int rank_final;   // push AG: publish the final unit rank-level (cta_signal_rank); flat calls only (a
                    //   per-call SPMD-uniform choice: hierarchical phases may chain on some ranks only)
  int chain;        // 1: first launch of a chained pair (publishes per-CTA completion), 2: second (waits for it
                    //    instead of the PDL grid-completion wait); see "chained launches" below
  int64_t item;     // direct kernels: units per dynamically claimed work item (0: static CTA slices)
  int64_t timeout_ns;
  int64_t blk;              // units per sub-block
  int64_t sub_stride;       // stride between sub-blocks (shared layout)
  int64_t istride;          // stride between members' blocks / chunks
  int64_t send_sub_stride;  // AG: sub-block stride inside send (contiguous: blk)
  int64_t out_sub_stride;   // RS: sub-block stride inside the final output
  int64_t base[PCCL_MAXR];  // per row: layout base offset (group-uniform)
  uint64_t epoch[PCCL_MAXR];
  uint32_t slot_off[PCCL_MAXR];  // per row: flag slot offset in words
  uint32_t chain_slot_off[PCCL_MAXR];  // chain == 1, per row: slot of the second launch's group
  uint32_t meta[PCCL_MAXR];      // per row: call-signature hash
  int8_t row_rank[PCCL_MAXR];
  int8_t grank[PCCL_MAXR];
  int8_t gmem[PCCL_MAXR][PCCL_MAXR];  // per row: world ranks of the group
  uint64_t *flags[PCCL_MAXR];         // per world rank: flag arena
  char *send[PCCL_MAXR];              // per world rank
  char *recv[PCCL_MAXR];
  char *work[PCCL_MAXR];
  char *out[PCCL_MAXR];
  volatile int *err;                  // host-mapped error word
  uint64_t *trace;                    // optional: per (row, cta) event log, PCCL_TRACE_EVENTS words
};

#define PCCL_TRACE_EVENTS 128
#define PCCL_TRACE_LAUNCHES 8
enum TraceKind { TR_START = 1, TR_WAIT = 2, TR_SIGNAL = 3, TR_END = 4, TR_EXIT = 5, TR_RESIDENT = 6, TR_EPILOGUE = 7, TR_PDL = 8 };

// --------------------------------------------------------------------------
// memory-model primitives
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ volatile uint64_t *err_mirror(const LaunchParams &P, int r) {
  return P.flags[r] + PCCL_WCTRL_OFF + PCCL_WCTRL_ERR;
}

struct Ctx {
  const LaunchParams *P;
  int y;   // launch row
  int r;   // world rank
  int gi;  // index in group
  int gs;
  int b;   // CTA index in row
  uint64_t epoch;
  uint64_t *my_slot;
  uint64_t t0;
  uint64_t *tr;  // trace cursor base (nullptr: tracing off)
  int ntr;
  uint32_t ll_peers;  // LL kernels: world ranks whose channel counter the last CTA advances
  int ll_ctr;         // WCTRL index of those counters: 0 (LL) or PCCL_WCTRL_LL128
  uint64_t chain_epoch;  // chain == 1: the second launch's epoch (published per CTA at exit)

  __device__ __forceinline__ int world(int m) const { return P->gmem[y][m]; }
  __device__ __forceinline__ uint64_t *slot_in(int m) const {
    return P->flags[world(m)] + P->slot_off[y];
  }
  static __device__ __forceinline__ uint64_t *word(uint64_t *slot, int kind, int src, int cta) {
    return slot + ((size_t)(kind * PCCL_MAXR + src) * PCCL_MAX_CTAS + cta);
  }
};

// Programmatic dependent launch: let the next collective's grid be scheduled
// while this one drains, and wait for the previous grid's completion (and
// memory flush) before touching anything. No-ops without the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Chained launches (hierarchical collectives, real mode): the two phases are
// two launches on one stream with programmatic dependent launch. The second
// does NOT wait for the first grid's completion (griddepcontrol.wait): its
// CTA b waits only for CTA b of the first launch, which publishes, when it
// exits, the second launch's epoch in the ITEM word [PCCL_MAXR - 1][b] of the
// second group's slot in its own arena (st.release.gpu after a CTA barrier).
// Both launches cut the element range into the same CTA slices (same grid,
// same unit size: the host chains only 16-byte-aligned layouts), and the
// second phase touches nothing of the first but that slice, so the phase
// boundary costs no grid drain and no relaunch. The first launch's own
// griddepcontrol.wait still orders the pair after everything before it.
__device__ __forceinline__ uint64_t *chain_word(const LaunchParams &P, int r, uint32_t slot_off, int b) {
  return P.flags[r] + slot_off + ((size_t)(F_ITEM * PCCL_MAXR + (PCCL_MAXR - 1)) * PCCL_MAX_CTAS + b);
}
__device__ __forceinline__ void st_release_gpu(uint64_t *p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ Ctx make_ctx(const LaunchParams &P) {
  const uint64_t t_resident = P.trace ? global_timer_ns() : 0;  // CTA scheduled (before the PDL wait)
  if (P.chain != 2) pdl_wait();
  const uint64_t t_pdl = P.trace ? global_timer_ns() : 0;  // the previous grid is complete
  pdl_launch_dependents();
  Ctx c;
  c.P = &P;
  c.y = blockIdx.y;
  c.r = P.row_rank[c.y];
  c.gi = P.grank[c.y];
  c.gs = P.gs;
  c.b = blockIdx.x;
  c.my_slot = P.flags[c.r] + P.slot_off[c.y];
  // The group's epoch lives in device memory (CTRL[0] of my slot): read it at
  // launch, the last CTA to exit advances it. No host bookkeeping, so a
  // captured CUDA graph replays correctly.
  c.epoch = *reinterpret_cast<volatile uint64_t *>(c.my_slot + PCCL_CTRL_OFF) + 1;
  c.t0 = global_timer_ns();
  c.tr = P.trace ? P.trace + ((size_t)c.y * P.ctas + c.b) * PCCL_TRACE_EVENTS : nullptr;
  c.ntr = 0;
  c.ll_peers = 0;
  c.ll_ctr = 0;
  c.chain_epoch = 0;
  if (P.chain == 1)
    c.chain_epoch = *reinterpret_cast<volatile uint64_t *>(P.flags[c.r] + P.chain_slot_off[c.y] + PCCL_CTRL_OFF) + 1;
  if (P.chain == 2) {  // wait for CTA b of the first launch (its slice of the first phase is complete)
    __shared__ int s_chain;
    if (threadIdx.x == 0) {
      const uint64_t *w = chain_word(P, c.r, P.slot_off[c.y], c.b);
      int code = 0;
      uint32_t it = 0;
      while (true) {
        uint64_t v;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
        if (v >= c.epoch) break;
        if ((++it & 4095u) == 0) {  // rare host-memory reads: the first phase usually takes tens of us
          if (const uint64_t e = *err_mirror(P, c.r)) { code = (int)e; break; }
          if (global_timer_ns() - c.t0 > (uint64_t)P.timeout_ns) { code = 5; break; }  // PCCL_ERR_TIMEOUT
        }
      }
      if (code) {  // the body's first wait then sees the error
        *err_mirror(P, c.r) = (uint64_t)code;
        if (*P.err == 0) *P.err = code;
      }
      s_chain = code;
    }
    __syncthreads();
  }
  if (c.tr && threadIdx.x == 0) {
    c.tr[c.ntr++] = (t_resident << 16) | (TR_RESIDENT << 12);
    c.tr[c.ntr++] = (t_pdl << 16) | (TR_PDL << 12);
    c.tr[c.ntr++] = (c.t0 << 16) | (TR_START << 12);
  }
  return c;
}

// Runs when a kernel returns (any path): the last CTA of the row to leave
// publishes the epoch for the next launch on this stream.
struct CtaEpilogue {
  Ctx &c;
  __device__ explicit CtaEpilogue(Ctx &cc) : c(cc) {}
  __device__ ~CtaEpilogue() {
    if (c.P->chain == 1) {  // this CTA's slice of the first phase is complete: release the second launch's CTA b
      // (no check of the host-mapped error word here: 128 CTAs reading host
      // memory at once stalled the exits by up to 120 us; a failed first phase
      // has set the error word, which the second phase's waits observe)
      __syncthreads();
      if (threadIdx.x == 0) st_release_gpu(chain_word(*c.P, c.r, c.P->chain_slot_off[c.y], c.b), c.chain_epoch);
    }
    if (c.tr && threadIdx.x == 0 && c.ntr < PCCL_TRACE_EVENTS)
      c.tr[c.ntr++] = (global_timer_ns() << 16) | ((uint64_t)TR_EXIT << 12);
    if (threadIdx.x == 0) {
      unsigned long long *ctrl = reinterpret_cast<unsigned long long *>(c.my_slot + PCCL_CTRL_OFF);
      const unsigned long long old = atomicAdd(ctrl + 1, 1ull);
      if (old == (unsigned long long)(c.P->ctas - 1)) {
        ctrl[1] = 0;
        for (int k = 2; k <= 10; ++k) ctrl[k] = 0;  // work-item counters (every CTA's last claim returned before it got here)
        *reinterpret_cast<volatile unsigned long long *>(ctrl) = c.epoch;
        if (c.ll_peers) {
          volatile uint64_t *lc = c.P->flags[c.r] + PCCL_WCTRL_OFF;
          for (int q = 0; q < PCCL_MAXR; ++q)
            if ((c.ll_peers >> q) & 1u) lc[c.ll_ctr + q] = lc[c.ll_ctr + q] + 1;
        }
      }
      if (c.tr && c.ntr < PCCL_TRACE_EVENTS) c.tr[c.ntr++] = (global_timer_ns() << 16) | ((uint64_t)TR_EPILOGUE << 12);
    }
  }
};

// thread 0 only: append (time, kind, unit) to this CTA's trace
__device__ __forceinline__ void trace_ev(Ctx &c, int kind, int unit) {
  if (c.tr && threadIdx.x == 0 && c.ntr < PCCL_TRACE_EVENTS)
    c.tr[c.ntr++] = (global_timer_ns() << 16) | ((uint64_t)kind << 12) | (uint64_t)(unit & 0xfff);
}

// Flood ABORT into every member's slot (all sources, all CTAs) so that every
// waiter of this group, on every GPU, wakes up. Called by a whole CTA.
__device__ __noinline__ void abort_group(const Ctx &c, int code) {
  if (threadIdx.x == 0 && *c.P->err == 0) {  // error path only: reading host memory is fine here
    *c.P->err = code;  // host-visible (the host reports it)
    __threadfence_system();
  }
  if (threadIdx.x < c.gs)  // every member's device mirror: its spinning CTAs stop without host-memory reads
    st_relaxed_sys(const_cast<uint64_t *>(err_mirror(*c.P, c.world(threadIdx.x))), (uint64_t)code);
  const uint64_t v = PCCL_ABORT_BIT | (uint64_t)code;
  const int per_member = 4 * PCCL_MAXR * PCCL_MAX_CTAS;  // READY, DONE, META (copy-engine waits), ITEM
  for (int m = 0; m < c.gs; ++m) {
    uint64_t *slot = c.slot_in(m);
    for (int i = threadIdx.x; i < per_member; i += blockDim.x) st_relaxed_sys(slot + i, v);
  }
  __threadfence_system();
}

// Spin (one thread) until word >= target. Returns 0 or an error code.
__device__ __forceinline__ int spin_ge(const Ctx &c, const uint64_t *w, uint64_t target) {
  uint32_t it = 0;
  while (true) {
    uint64_t v = ld_acquire_sys(w);
    if (v & PCCL_ABORT_BIT) return (int)(v & 0xff);
    if (v >= target) return 0;
    if ((++it & 255u) == 0) {
      if (const uint64_t e = *err_mirror(*c.P, c.r)) return (int)e;
      if (global_timer_ns() - c.t0 > (uint64_t)c.P->timeout_ns) return 5;  // PCCL_ERR_TIMEOUT
    }
  }
}

// Step-structure helpers shared by the kernels and pccl_schedule (host).
__host__ __device__ __forceinline__ int ring_prev(int gi, int gs) { return (gi - 1 + gs) % gs; }
__host__ __device__ __forceinline__ int ring_next(int gi, int gs) { return (gi + 1) % gs; }
// recursive doubling AG, step k (collectives.py:121-124)
__host__ __device__ __forceinline__ int recdbl_partner(int gi, int k) { return gi ^ (1 << k); }
// recursive halving RS, step k (collectives.py:151-153)
__host__ __device__ __forceinline__ int rechalf_partner(int gi, int gs, int k) { return gi ^ (gs >> (k + 1)); }

// READY word: epoch << 32 | (call-signature hash & 0x3fffff) << 10 | (unit + 1).
// Folding the signature into the progress word makes the cross-rank check
// free: no separate META store (and no extra fence) on the entry handshake.
__device__ __forceinline__ uint64_t ready_value(const Ctx &c, int unit) {
  return (c.epoch << 32) | ((uint64_t)(c.P->meta[c.y] & 0x3fffffu) << 10) | (uint64_t)(unit + 1);
}
// 0 = satisfied, > 0 = error code, -1 = not yet. A later epoch satisfies any
// wait of an earlier one (the writer already published everything of ours).
__device__ __forceinline__ int ready_check(const Ctx &c, uint64_t v, int unit) {
  if (v & PCCL_ABORT_BIT) return (int)(v & 0xff);
  const uint64_t ep = (v >> 32) & 0x7fffffffull;
  if (ep > c.epoch) return 0;
  if (ep < c.epoch) return -1;
  if (((v >> 10) & 0x3fffffu) != (c.P->meta[c.y] & 0x3fffffu)) {
    // diagnostics for pccl_world_error_detail: first mismatch only
    if (atomicCAS((int *)&c.P->err[8], 0, 1) == 0) {
      c.P->err[9] = (int)c.epoch;
      c.P->err[10] = (int)(c.P->meta[c.y] & 0x3fffffu);
      c.P->err[11] = (int)((v >> 10) & 0x3fffffu);
      c.P->err[12] = c.r;
      c.P->err[13] = unit;
      c.P->err[14] = (int)(v & 0x3ffu);
      c.P->err[15] = c.b;
    }
    return 4;  // PCCL_ERR_LENGTH_MISMATCH
  }
  return (v & 0x3ffu) >= (uint64_t)(unit + 1) ? 0 : -1;
}
__device__ __forceinline__ int spin_ready(const Ctx &c, const uint64_t *w, int unit) {
  uint32_t it = 0;
  while (true) {
    const int r = ready_check(c, ld_acquire_sys(w), unit);
    if (r >= 0) return r;
    if ((++it & 255u) == 0) {
      if (const uint64_t e = *err_mirror(*c.P, c.r)) return (int)e;
      if (global_timer_ns() - c.t0 > (uint64_t)c.P->timeout_ns) return 5;  // PCCL_ERR_TIMEOUT
    }
  }
}

// CTA-wide: wait until member m has completed `unit` (its call signature is
// verified on every wait). Returns false (after aborting the group) on error.
__device__ __forceinline__ bool cta_wait(Ctx &c, int m, int unit) {
  int code = 0;
  if (threadIdx.x == 0) code = spin_ready(c, Ctx::word(c.my_slot, F_READY, m, c.b), unit);
  int ok = __syncthreads_and(code == 0);
  if (!ok) {
    __shared__ int s_code;
    if (threadIdx.x == 0) s_code = code;
    __syncthreads();
    if (s_code != 0) abort_group(c, s_code);
    return false;
  }
  trace_ev(c, TR_WAIT, unit);
  return true;
}

// CTA-wide: wait for every member in `mask` (bit m) to complete `unit`.
// `idx`: the writers' CTA index whose words to wait on (default: mine).
__device__ __forceinline__ bool cta_wait_mask(Ctx &c, uint32_t mask, int unit, int idx = -1) {
  int code = 0;
  const int m = threadIdx.x;
  if (m < c.gs && ((mask >> m) & 1u)) code = spin_ready(c, Ctx::word(c.my_slot, F_READY, m, idx < 0 ? c.b : idx), unit);
  int ok = __syncthreads_and(code == 0);
  if (!ok) {
    __shared__ int s_code;
    if (threadIdx.x == 0) s_code = 0;
    __syncthreads();
    if (code != 0) atomicCAS(&s_code, 0, code);
    __syncthreads();
    abort_group(c, s_code ? s_code : 5);
    return false;
  }
  trace_ev(c, TR_WAIT, unit);
  return true;
}

// CTA-wide: publish completion of `unit` to member m (after a CTA barrier so
// every thread's stores of the unit are ordered before the release).
__device__ __forceinline__ void cta_signal(Ctx &c, int m, int unit) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_sys(Ctx::word(c.slot_in(m), F_READY, c.gi, c.b), ready_value(c, unit));
  trace_ev(c, TR_SIGNAL, unit);
}
__device__ __forceinline__ void cta_signal_mask(Ctx &c, uint32_t mask, int unit) {
  __syncthreads();
  const int m = threadIdx.x;
  if (m < c.gs && ((mask >> m) & 1u))
    st_release_sys(Ctx::word(c.slot_in(m), F_READY, c.gi, c.b), ready_value(c, unit));
  trace_ev(c, TR_SIGNAL, unit);
}
// Rank-level publish of a push kernel's FINAL unit: every CTA releases its
// stores at gpu scope into a counter in my slot (CTRL[11]) and the row's last
// CTA publishes once per member with a system-scope release into the word of
// CTA 0 (the acq_rel RMW chain + the CTA barrier make that release
// cumulative over every CTA's stores). One MEMBAR.SYS per rank instead of
// one per CTA and member: 128 CTAs issuing system fences at once cost
// ~4-5 us (profiles/r2_launch_boundary.md). Waiters use cta_wait_mask(...,
// idx = 0). For a final unit only: a receiver now waits for all of a
// sender's CTAs, which a pipelined step cannot afford.
__device__ __forceinline__ void cta_signal_rank(Ctx &c, uint32_t mask, int unit) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(c.my_slot + PCCL_CTRL_OFF) + 11;
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
    s_last = old == (unsigned long long)(c.P->ctas - 1);
    if (s_last) *reinterpret_cast<volatile unsigned long long *>(ctr) = 0;  // next launch: after this grid
  }
  __syncthreads();
  const int m = threadIdx.x;
  if (s_last && m < c.gs && ((mask >> m) & 1u))
    st_release_sys(Ctx::word(c.slot_in(m), F_READY, c.gi, 0), ready_value(c, unit));
  trace_ev(c, TR_SIGNAL, unit);
}
// Pull kernels publish data that lives in the writer's OWN memory: once a
// gpu-scope fence has made it visible at the writer's L2 (the point of
// coherence every NVLink reader goes through), a relaxed system-scope flag
// store suffices. MEMBAR.GPU costs a local L2 round trip instead of the
// system-wide drain of MEMBAR.SYS. Entry signals (data written before the
// launch) and exit signals (my remote loads have returned) need no fence.
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void cta_signal_local(Ctx &c, int m, int unit) {
  if (!c.P->local_fence) { cta_signal(c, m, unit); return; }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_gpu();
    st_relaxed_sys(Ctx::word(c.slot_in(m), F_READY, c.gi, c.b), ready_value(c, unit));
  }
  trace_ev(c, TR_SIGNAL, unit);
}
__device__ __forceinline__ void cta_signal_entry(Ctx &c, uint32_t mask, int unit = 0) {
  if (!c.P->local_fence) { cta_signal_mask(c, mask, unit); return; }
  const int m = threadIdx.x;
  if (m < c.gs && ((mask >> m) & 1u)) st_relaxed_sys(Ctx::word(c.slot_in(m), F_READY, c.gi, c.b), ready_value(c, unit));
  trace_ev(c, TR_SIGNAL, unit);
}

// Exit barrier: tell every member in `to` that this CTA has finished reading
// their buffers; wait until every member in `from` has finished reading ours.
__device__ __forceinline__ bool cta_exit(Ctx &c, uint32_t to, uint32_t from) {
  if (c.P->skip_exit) return true;
  __syncthreads();
  const int m = threadIdx.x;
  if (m < c.gs && ((to >> m) & 1u)) {
    if (c.P->local_fence) st_relaxed_sys(Ctx::word(c.slot_in(m), F_DONE, c.gi, c.b), c.epoch);
    else st_release_sys(Ctx::word(c.slot_in(m), F_DONE, c.gi, c.b), c.epoch);
  }
  int code = 0;
  if (m < c.gs && ((from >> m) & 1u)) code = spin_ge(c, Ctx::word(c.my_slot, F_DONE, m, c.b), c.epoch);
  int ok = __syncthreads_and(code == 0);
  if (!ok) {
    __shared__ int s_code;
    if (threadIdx.x == 0) s_code = 0;
    __syncthreads();
    if (code != 0) atomicCAS(&s_code, 0, code);
    __syncthreads();
    abort_group(c, s_code ? s_code : 5);
    return false;
  }
  trace_ev(c, TR_END, 0);
  return true;
}

// --------------------------------------------------------------------------
// LL protocol (small direct collectives): flags travel inside the data.
// Every 16-byte store carries 8 payload bytes and two copies of a 32-bit tag,
// {d0, tag, d1, tag}; each 8-byte half is single-copy atomic over NVLink, so a
// reader that sees both tags equal to the expected value holds valid payload.
// A (src -> dst) channel alternates two message regions in dst's arena by the
// parity of its message count (kept per peer in each rank's WCTRL words, and
// advanced by the last CTA of every LL launch). Direct collectives are
// all-to-all, so src starts message s+2 only after a collective in which dst
// sent to src after dst had consumed message s: a region is never rewritten
// before it was read. No entry handshake, no fence, no exit barrier; user
// buffers are only touched locally. A 16-byte header {hash, tag, hash, tag}
// per message carries the call signature (cross-rank mismatch -> LengthMismatch).
// --------------------------------------------------------------------------
__device__ __forceinline__ char *ll_region(const LaunchParams &P, int dst, uint32_t tag, int src) {
  return reinterpret_cast<char *>(P.flags[dst] + PCCL_LL_OFF) +
         ((size_t)(tag & 1u) * PCCL_MAXR + src) * PCCL_LL_REGION_BYTES;
}
__device__ __forceinline__ char *ll128_region(const LaunchParams &P, int dst, uint32_t tag, int src) {
  return reinterpret_cast<char *>(P.flags[dst]) + PCCL_LL128_OFF +
         ((size_t)(tag & 1u) * PCCL_MAXR + src) * PCCL_LL128_REGION_BYTES;
}
// the message region of a channel in the launch's format (Ctx::ll_ctr)
__device__ __forceinline__ char *ll_region_of(const Ctx &c, int dst, uint32_t tag, int src) {
  return c.ll_ctr ? ll128_region(*c.P, dst, tag, src) : ll_region(*c.P, dst, tag, src);
}
__device__ __forceinline__ void ll_st(uint4 *p, uint32_t a, uint32_t b, uint32_t tag) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(tag), "r"(b), "r"(tag)
               : "memory");
}
__device__ __forceinline__ uint4 ll_ld(const uint4 *p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ bool ll_ok(const uint4 &v, uint32_t tag) { return v.y == tag && v.w == tag; }
// Spin until both tags match. Returns 0, or an error code: the world error,
// 5 on timeout, 4 when the sender's header shows another call signature
// (checked on the slow path only, so a mismatched count cannot hang us).
__device__ __forceinline__ int ll_wait(const Ctx &c, const uint4 *p, uint32_t tag, uint4 &v, const uint4 *hdr) {
  uint32_t it = 0;
  while (true) {
    v = ll_ld(p);
    if (ll_ok(v, tag)) return 0;
    if ((++it & 1023u) == 0) {
      if (const uint64_t e = *err_mirror(*c.P, c.r)) return (int)e;
      const uint4 h = ll_ld(hdr);
      if (ll_ok(h, tag) && (h.x != c.P->meta[c.y] || h.z != c.P->meta[c.y])) return 4;
      if (global_timer_ns() - c.t0 > (uint64_t)c.P->timeout_ns) return 5;
    }
  }
}
// Per group member m: the tag of this launch's message on channel (me, m).
__device__ __forceinline__ void ll_tags(Ctx &c, uint32_t *s_tag) {
  volatile const uint64_t *lc = c.P->flags[c.r] + PCCL_WCTRL_OFF;
  if (threadIdx.x < c.gs) {
    const uint64_t n = lc[c.ll_ctr + c.world(threadIdx.x)] + 1;
    s_tag[threadIdx.x] = (uint32_t)n ? (uint32_t)n : 1u;  // never 0 (cleared memory)
  }
  for (int m = 0; m < c.gs; ++m)
    if (m != c.gi) c.ll_peers |= 1u << c.world(m);
  __syncthreads();
}
// CTA 0: post the signature header of my message to every member.
__device__ __forceinline__ void ll_post_headers(const Ctx &c, const uint32_t *s_tag) {
  const int m = threadIdx.x;
  if (c.b == 0 && m < c.gs && m != c.gi) {
    const uint32_t meta = c.P->meta[c.y];
    ll_st(reinterpret_cast<uint4 *>(ll_region_of(c, c.world(m), s_tag[m], c.r)), meta, meta, s_tag[m]);
  }
}
// CTA-wide, after the data: every member's header carries my signature.
// `code` is this thread's error from the data phase (0 if none).
__device__ __forceinline__ bool ll_finish(Ctx &c, const uint32_t *s_tag, int code) {
  const int m = threadIdx.x;
  if (code == 0 && m < c.gs && m != c.gi) {
    uint4 v;
    const uint4 *h = reinterpret_cast<const uint4 *>(ll_region_of(c, c.r, s_tag[m], c.world(m)));
    code = ll_wait(c, h, s_tag[m], v, h);
    if (code == 0 && (v.x != c.P->meta[c.y] || v.z != c.P->meta[c.y])) code = 4;
    if (code == 4 && atomicCAS((int *)&c.P->err[8], 0, 1) == 0) {
      c.P->err[9] = (int)c.epoch;
      c.P->err[10] = (int)(c.P->meta[c.y] & 0x3fffffu);
      c.P->err[11] = (int)(v.x & 0x3fffffu);
      c.P->err[12] = c.r;
      c.P->err[13] = -1;
      c.P->err[14] = c.world(m);
      c.P->err[15] = c.b;
    }
  }
  if (__syncthreads_and(code == 0)) {
    trace_ev(c, TR_END, 0);
    return true;
  }
  __shared__ int s_code;
  if (threadIdx.x == 0) s_code = 0;
  __syncthreads();
  if (code != 0) atomicCAS(&s_code, 0, code);
  __syncthreads();
  abort_group(c, s_code ? s_code : 5);
  return false;
}

// --------------------------------------------------------------------------
// slicing: CTA b of C owns [lo,hi) of every sub-block; sub-slice t of nsub
// --------------------------------------------------------------------------
__device__ __forceinline__ void split32(int64_t len, int parts, int idx, int64_t &lo, int64_t &hi) {
  const int64_t n32 = (len + 31) / 32;
  lo = (n32 * idx / parts) * 32;
  hi = (n32 * (idx + 1) / parts) * 32;
  if (lo > len) lo = len;
  if (hi > len) hi = len;
}
__device__ __forceinline__ void cta_subslice(const Ctx &c, int t, int64_t &lo, int64_t &hi) {
  int64_t a, e;
  split32(c.P->blk, c.P->ctas, c.b, a, e);
  int64_t sa, se;
  split32(e - a, c.P->nsub, t, sa, se);
  lo = a + sa;
  hi = a + se;
}

// Dynamic work distribution for the single-step (direct) kernels. Measured
// with tools/trace.py at p=4, 128 MiB: with static CTA slices the CTAs'
// finishing times spread over ~40 us (push AG: 108..149 us) because NVLink
// arbitration is not fair between SMs, and the link idles in the tail.
// Instead every CTA claims items from a per-row counter in its own slot
// (CTRL[2], local atomics; the row's last CTA resets it in CtaEpilogue), and
// prefetches its next claim while moving the current item. The flag protocol
// is unchanged: CTA b still signals / waits on the peers' CTA b, and since a
// rank's kernel completes only after all of its CTAs' waits, the union over
// b still covers every item of every peer — which is enough only where the
// moved data is consumed after the launch (AG push) or was ready before it
// (pull reads of the peers' inputs). Data pushed and consumed inside one
// launch (RS direct push: push, then fold) keeps static slices.
template <typename F>
__device__ __forceinline__ void for_items(const Ctx &c, int64_t total, F &&body, int ctr_word = 2) {
  __shared__ long long s_item[2];
  unsigned long long *ctr = reinterpret_cast<unsigned long long *>(c.my_slot + PCCL_CTRL_OFF + ctr_word);
  if (threadIdx.x == 0) s_item[0] = (long long)atomicAdd(ctr, 1ull);
  __syncthreads();
  long long cur = s_item[0];
  for (int k = 1; cur < total; ++k) {
    unsigned long long nx = 0;
    if (threadIdx.x == 0) nx = atomicAdd(ctr, 1ull);  // in flight while this item moves
    body((int64_t)cur);
    if (threadIdx.x == 0) s_item[k & 1] = (long long)nx;
    __syncthreads();
    cur = s_item[k & 1];
  }
}

// Item-level progress (multi-step item kernels): member m's item i reached
// `unit` — F_ITEM[m][i] in the reader's arena. CTA-wide wait; returns false
// after aborting the group.
__device__ __forceinline__ bool item_wait(Ctx &c, int m, int item, int unit) {
  int code = 0;
  if (threadIdx.x == 0) code = spin_ready(c, Ctx::word(c.my_slot, F_ITEM, m, item), unit);
  if (!__syncthreads_and(code == 0)) {
    __shared__ int s_code;
    if (threadIdx.x == 0) s_code = code;
    __syncthreads();
    if (s_code != 0) abort_group(c, s_code);
    return false;
  }
  return true;
}
// Publish item `item` at `unit` to member m and to myself (local dependency
// of the next step), after a CTA barrier. The data is in my own memory (pull
// kernels), so the local_fence publish applies (see cta_signal_local).
__device__ __forceinline__ void item_signal(Ctx &c, int m, int item, int unit) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t v = ready_value(c, unit);
    if (c.P->local_fence) {
      fence_gpu();
      st_relaxed_sys(Ctx::word(c.slot_in(m), F_ITEM, c.gi, item), v);
    } else {
      st_release_sys(Ctx::word(c.slot_in(m), F_ITEM, c.gi, item), v);
    }
    st_relaxed_sys(Ctx::word(c.my_slot, F_ITEM, c.gi, item), v);
  }
}

// --------------------------------------------------------------------------
// unit types and loads
// --------------------------------------------------------------------------
template <int U> struct VecT;
template <> struct VecT<16> { using T = uint4; };
template <> struct VecT<8> { using T = uint2; };
template <> struct VecT<4> { using T = unsigned int; };
template <> struct VecT<2> { using T = unsigned short; };
template <> struct VecT<1> { using T = unsigned char; };

// Peer data is read with .cg (L2-coherent, no L1 allocation): it is produced
// during this kernel by another GPU and published through the flag protocol.
template <typename T> __device__ __forceinline__ T ld_peer(const T *p) { return __ldcg(p); }

// Every iteration keeps UNROLL independent loads in flight per thread, also
// for the last partial iteration (predicated), so short slices do not fall
// back to one outstanding load per thread.
template <int U, int UNROLL>
__device__ __forceinline__ void copy_units(char *dst, const char *src, int64_t lo, int64_t hi) {
  using T = typename VecT<U>::T;
  T *d = reinterpret_cast<T *>(dst);
  const T *s = reinterpret_cast<const T *>(src);
  const int nt = blockDim.x;
  for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)UNROLL * nt) {
    T v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (i + (int64_t)u * nt < hi) v[u] = ld_peer(s + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (i + (int64_t)u * nt < hi) d[i + (int64_t)u * nt] = v[u];
  }
}

// copy_units that also writes a second destination from the same loads (a
// push all-gather storing my block into a peer and into my own output: one
// read of the send buffer, no separate local-copy pass in the tail).
template <int U, int UNROLL>
__device__ __forceinline__ void copy_units_dup(char *dst, char *dst2, const char *src, int64_t lo, int64_t hi) {
  using T = typename VecT<U>::T;
  T *d = reinterpret_cast<T *>(dst);
  T *d2 = reinterpret_cast<T *>(dst2);
  const T *s = reinterpret_cast<const T *>(src);
  const int nt = blockDim.x;
  for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)UNROLL * nt) {
    T v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (i + (int64_t)u * nt < hi) v[u] = ld_peer(s + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (i + (int64_t)u * nt < hi) d[i + (int64_t)u * nt] = v[u];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (i + (int64_t)u * nt < hi) d2[i + (int64_t)u * nt] = v[u];
  }
}

// --------------------------------------------------------------------------
// reduction units: VEC -> one uint4 (4 fp32 or 8 bf16/f16), else one element.
// Accumulation is always fp32 with explicit round-to-nearest adds (no
// reassociation, no contraction): the fold order is the algorithm's.
// --------------------------------------------------------------------------
template <int DT, bool VEC> struct RUnit;

template <> struct RUnit<DT_F32, true> {
  using T = uint4;
  static constexpr int N = 4;
  struct Acc { float v[4]; };
  static __device__ __forceinline__ Acc load(T u) {
    Acc a; a.v[0] = __uint_as_float(u.x); a.v[1] = __uint_as_float(u.y);
    a.v[2] = __uint_as_float(u.z); a.v[3] = __uint_as_float(u.w); return a;
  }
  static __device__ __forceinline__ T store(const Acc &a) {
    return make_uint4(__float_as_uint(a.v[0]), __float_as_uint(a.v[1]), __float_as_uint(a.v[2]),
                      __float_as_uint(a.v[3]));
  }
};
template <> struct RUnit<DT_F32, false> {
  using T = unsigned int;
  static constexpr int N = 1;
  struct Acc { float v[1]; };
  static __device__ __forceinline__ Acc load(T u) { Acc a; a.v[0] = __uint_as_float(u); return a; }
  static __device__ __forceinline__ T store(const Acc &a) { return __float_as_uint(a.v[0]); }
};

__device__ __forceinline__ float2 bf2_to_f2(unsigned x) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162 *>(&x);
  return __bfloat1622float2(h);
}
__device__ __forceinline__ unsigned f2_to_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<unsigned *>(&h);
}
__device__ __forceinline__ float2 h2_to_f2(unsigned x) {
  __half2 h = *reinterpret_cast<__half2 *>(&x);
  return __half22float2(h);
}
__device__ __forceinline__ unsigned f2_to_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<unsigned *>(&h);
}

template <> struct RUnit<DT_BF16, true> {
  using T = uint4;
  static constexpr int N = 8;
  struct Acc { float v[8]; };
  static __device__ __forceinline__ Acc load(T u) {
    Acc a; float2 f;
    f = bf2_to_f2(u.x); a.v[0] = f.x; a.v[1] = f.y;
    f = bf2_to_f2(u.y); a.v[2] = f.x; a.v[3] = f.y;
    f = bf2_to_f2(u.z); a.v[4] = f.x; a.v[5] = f.y;
    f = bf2_to_f2(u.w); a.v[6] = f.x; a.v[7] = f.y;
    return a;
  }
  static __device__ __forceinline__ T store(const Acc &a) {
    return make_uint4(f2_to_bf2(a.v[0], a.v[1]), f2_to_bf2(a.v[2], a.v[3]), f2_to_bf2(a.v[4], a.v[5]),
                      f2_to_bf2(a.v[6], a.v[7]));
  }
};
template <> struct RUnit<DT_BF16, false> {
  using T = unsigned short;
  static constexpr int N = 1;
  struct Acc { float v[1]; };
  static __device__ __forceinline__ Acc load(T u) { Acc a; a.v[0] = __uint_as_float(((unsigned)u) << 16); return a; }
  static __device__ __forceinline__ T store(const Acc &a) {
    __nv_bfloat16 h = __float2bfloat16_rn(a.v[0]);
    return *reinterpret_cast<unsigned short *>(&h);
  }
};
template <> struct RUnit<DT_F16, true> {
  using T = uint4;
  static constexpr int N = 8;
  struct Acc { float v[8]; };
  static __device__ __forceinline__ Acc load(T u) {
    Acc a; float2 f;
    f = h2_to_f2(u.x); a.v[0] = f.x; a.v[1] = f.y;
    f = h2_to_f2(u.y); a.v[2] = f.x; a.v[3] = f.y;
    f = h2_to_f2(u.z); a.v[4] = f.x; a.v[5] = f.y;
    f = h2_to_f2(u.w); a.v[6] = f.x; a.v[7] = f.y;
    return a;
  }
  static __device__ __forceinline__ T store(const Acc &a) {
    return make_uint4(f2_to_h2(a.v[0], a.v[1]), f2_to_h2(a.v[2], a.v[3]), f2_to_h2(a.v[4], a.v[5]),
                      f2_to_h2(a.v[6], a.v[7]));
  }
};
template <> struct RUnit<DT_F16, false> {
  using T = unsigned short;
  static constexpr int N = 1;
  struct Acc { float v[1]; };
  static __device__ __forceinline__ Acc load(T u) {
    __half h = *reinterpret_cast<__half *>(&u);
    Acc a; a.v[0] = __half2float(h); return a;
  }
  static __device__ __forceinline__ T store(const Acc &a) {
    __half h = __float2half_rn(a.v[0]);
    return *reinterpret_cast<unsigned short *>(&h);
  }
};

template <typename Acc, int N>
__device__ __forceinline__ void acc_add(Acc &a, const Acc &b) {
#pragma unroll
  for (int i = 0; i < N; ++i) a.v[i] = __fadd_rn(a.v[i], b.v[i]);
}

// dst[i] = round(a[i] + b[i]) over units [lo,hi); a local, b peer.
template <int DT, bool VEC, int UNROLL>
__device__ __forceinline__ void reduce2_units(char *dst, const char *a, const char *b, int64_t lo, int64_t hi) {
  using R = RUnit<DT, VEC>;
  using T = typename R::T;
  T *d = reinterpret_cast<T *>(dst);
  const T *x = reinterpret_cast<const T *>(a);
  const T *y = reinterpret_cast<const T *>(b);
  const int nt = blockDim.x;
  for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)UNROLL * nt) {
    T vy[UNROLL], vx[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (i + (int64_t)u * nt < hi) vy[u] = ld_peer(y + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (i + (int64_t)u * nt < hi) vx[u] = __ldcg(x + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (i + (int64_t)u * nt < hi) {
        typename R::Acc sum = R::load(vx[u]);
        acc_add<typename R::Acc, R::N>(sum, R::load(vy[u]));
        d[i + (int64_t)u * nt] = R::store(sum);
      }
    }
  }
}


// --------------------------------------------------------------------------
// 256-bit global accesses (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256)
// --------------------------------------------------------------------------
struct alignas(32) V256 {
  uint32_t x[8];
};
__device__ __forceinline__ V256 ld256_cg(const V256 *p) {
  V256 v;
  asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.x[0]), "=r"(v.x[1]), "=r"(v.x[2]), "=r"(v.x[3]), "=r"(v.x[4]), "=r"(v.x[5]), "=r"(v.x[6]),
                 "=r"(v.x[7])
               : "l"(p));
  return v;
}
__device__ __forceinline__ V256 ld256_nc(const V256 *p) {
  V256 v;
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.x[0]), "=r"(v.x[1]), "=r"(v.x[2]), "=r"(v.x[3]), "=r"(v.x[4]), "=r"(v.x[5]), "=r"(v.x[6]),
                 "=r"(v.x[7])
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st256(V256 *p, const V256 &v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.x[0]), "r"(v.x[1]), "r"(v.x[2]),
               "r"(v.x[3]), "r"(v.x[4]), "r"(v.x[5]), "r"(v.x[6]), "r"(v.x[7])
               : "memory");
}

// --------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk) + mbarriers: one elected thread moves large
// tiles between global memory (local or NVLink-mapped peer) and shared memory
// with almost no instruction overhead, so a few SMs keep MBs in flight.
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tma_load(void *smem_dst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_store(void *gdst, const void *smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// A per-CTA ring of S shared-memory stages of T bytes driven by one thread.
struct TmaRing {
  char *buf;
  uint64_t *full;
  int S;
  uint32_t T;
  uint32_t n;  // tiles issued so far (stage = n % S, parity = (n / S) & 1)
};

// One thread: copy the concatenation of segments (dst[i] <- src[i], len[i]
// bytes, multiples of 16) through the ring, keeping S-1 tile loads in flight.
// Returns after every store has *completed* (safe to publish with a flag).
template <typename SegFn>
__device__ __forceinline__ void tma_copy_segments(TmaRing &R, int nseg, SegFn seg) {
  // flatten tiles lazily: walk segments with (i, off)
  int li = 0, si = 0;          // load cursor (segment, offset) / store cursor
  int64_t loff = 0, soff = 0;
  char *d; const char *s; int64_t len;
  auto next_tile = [&](int &i, int64_t &off, char *&dd, const char *&ss, uint32_t &bytes) -> bool {
    while (i < nseg) {
      seg(i, dd, ss, len);
      if (off < len) {
        { const int64_t rem = len - off; bytes = rem < (int64_t)R.T ? (uint32_t)rem : R.T; }
        dd += off;
        ss += off;
        off += bytes;
        return true;
      }
      ++i;
      off = 0;
    }
    return false;
  };
  const uint32_t base = R.n;
  uint32_t issued = 0, retired = 0;
  char *ld; const char *ls; uint32_t lb;
  // prologue
  while (issued < (uint32_t)R.S && next_tile(li, loff, ld, ls, lb)) {
    const uint32_t k = base + issued;
    uint64_t *bar = R.full + (k % R.S);
    mbar_expect_tx(bar, lb);
    tma_load(R.buf + (size_t)(k % R.S) * R.T, ls, lb, bar);
    ++issued;
  }
  while (retired < issued) {
    const uint32_t k = base + retired;
    const int st = k % R.S;
    mbar_wait(R.full + st, (k / R.S) & 1);
    char *sd; const char *ss2; uint32_t sb;
    next_tile(si, soff, sd, ss2, sb);
    tma_store(sd, R.buf + (size_t)st * R.T, sb);
    tma_commit();
    ++retired;
    if (next_tile(li, loff, ld, ls, lb)) {
      tma_wait_read_all();  // stage st free again
      const uint32_t k2 = base + issued;
      uint64_t *bar = R.full + (k2 % R.S);
      mbar_expect_tx(bar, lb);
      tma_load(R.buf + (size_t)(k2 % R.S) * R.T, ls, lb, bar);
      ++issued;
    }
  }
  R.n = base + issued;
  tma_wait_all();
  fence_proxy_async();
}

}  // namespace pccl
