// kernels.cuh — the collective kernels (sm_100a). All are pull-based: a rank
// reads its peers' symmetric buffers over NVLink/NVSwitch with 16-byte .cg
// loads and writes only its own HBM, so outputs never need to be registered
// and there is no staging hop. Reductions are fused into the peer-load loop.
//
// Step structure (checked against collkit.simnet.build_schedule through
// pccl_schedule, see step tables in host code):
//   AG direct     : 1 step, every rank pulls every peer's block.
//   AG ring       : collectives.py:55-76 — step s pulls block (r-s) from r-1.
//   AG recursive  : collectives.py:107-129 — step k pulls 2^k blocks from r^2^k.
//   RS direct     : 1 step, chunk r pulled from every peer, folded in the
//                   order of the named algorithm (bit-exact fp32).
//   RS ring       : collectives.py:79-104 — carry chain, one hop per step.
//   RS recursive  : collectives.py:132-165 — halving butterfly.
// Each CTA owns a contiguous slice of every block; inside a step the slice is
// cut into `nsub` sub-slices, and every sub-slice completion is published to
// the consumer of that step, so step s+1 of sub-slice t overlaps step s of
// sub-slice t+1 (no per-step bubble).
#pragma once
#include "device.cuh"

namespace pccl {

constexpr int kThreads = 512;
#ifndef PCCL_UNROLL
#define PCCL_UNROLL 8
#endif
constexpr int kUnroll = PCCL_UNROLL;

__device__ __forceinline__ int ilog2(int x) { return 31 - __clz(x); }

// ============================================================================
// all-gather
// ============================================================================
// Member i's block lives at recv + (base + i*istride + t*sub_stride) * U for
// sub-blocks t < nsubblk; my own contribution is send + t*send_sub_stride*U.
template <int U>
__device__ __forceinline__ char *ag_block(const LaunchParams &P, char *buf, int y, int i, int t) {
  return buf + (P.base[y] + (int64_t)i * P.istride + (int64_t)t * P.sub_stride) * U;
}

template <int U>
__device__ __forceinline__ void ag_local_copy(const Ctx &c, int64_t lo, int64_t hi) {
  const LaunchParams &P = *c.P;
  for (int t = 0; t < P.nsubblk; ++t)
    copy_units<U, kUnroll>(ag_block<U>(P, P.recv[c.r], c.y, c.gi, t), P.send[c.r] + (int64_t)t * P.send_sub_stride * U,
                           lo, hi);
}

template <int U>
__global__ void __launch_bounds__(kThreads) k_ag_direct(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const uint32_t peers = ((1u << c.gs) - 1) & ~(1u << c.gi);
  cta_signal_entry(c, peers);  // my send buffer is ready
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  if (P.local_copy) ag_local_copy<U>(c, lo, hi);
  if (P.item <= 0) {
    // shift pattern with per-peer entry waits (see k_ag_direct_push)
    for (int i = 1; i < c.gs; ++i) {
      const int q = (c.gi + i) % c.gs;
      if (!cta_wait(c, q, 0)) return;
      const char *src = P.send[c.world(q)];
      for (int t = 0; t < P.nsubblk; ++t)
        copy_units<U, kUnroll>(ag_block<U>(P, P.recv[c.r], c.y, q, t), src + (int64_t)t * P.send_sub_stride * U, lo, hi);
    }
    cta_exit(c, peers, peers);
    return;
  }
  if (!cta_wait_mask(c, peers, 0)) return;
  {
    // items (range j, sub-block t, source i), source fastest so that the
    // CTAs in flight spread over all peers
    const int nd = c.gs - 1;
    const int64_t nj = (P.blk + P.item - 1) / P.item;
    for_items(c, nj * nd * P.nsubblk, [&](int64_t id) {
      const int64_t j = id / (nd * P.nsubblk);
      const int rem = (int)(id - j * nd * P.nsubblk);
      const int q = (c.gi + 1 + rem % nd) % c.gs, t = rem / nd;
      const int64_t a = j * P.item, e = min(a + P.item, P.blk);
      copy_units<U, kUnroll>(ag_block<U>(P, P.recv[c.r], c.y, q, t),
                             P.send[c.world(q)] + (int64_t)t * P.send_sub_stride * U, a, e);
    });
  }
  cta_exit(c, peers, peers);
}

template <int U>
__global__ void __launch_bounds__(kThreads) k_ag_ring(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub;
  const int prev = ring_prev(c.gi, gs), next = ring_next(c.gi, gs);
  // step 0: own block into recv (the block the ring starts forwarding)
  for (int t = 0; t < nsub; ++t) {
    int64_t lo, hi;
    cta_subslice(c, t, lo, hi);
    if (P.local_copy) ag_local_copy<U>(c, lo, hi);
    cta_signal_local(c, next, t);
  }
  char *my = P.recv[c.r];
  const char *pv = P.recv[c.world(prev)];
  for (int s = 1; s < gs; ++s) {
    const int blk = (c.gi - s + gs) % gs;  // block received at reference step s-1
    for (int t = 0; t < nsub; ++t) {
      if (!cta_wait(c, prev, (s - 1) * nsub + t)) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int j = 0; j < P.nsubblk; ++j)
        copy_units<U, kUnroll>(ag_block<U>(P, my, c.y, blk, j), ag_block<U>(P, const_cast<char *>(pv), c.y, blk, j), lo,
                               hi);
      if (s < gs - 1) cta_signal_local(c, next, s * nsub + t);
    }
  }
  cta_exit(c, 1u << prev, 1u << next);
}

template <int U>
__global__ void __launch_bounds__(kThreads) k_ag_rec(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub, L = ilog2(gs);
  uint32_t partners = 0;
  for (int k = 0; k < L; ++k) partners |= 1u << recdbl_partner(c.gi, k);
  for (int t = 0; t < nsub; ++t) {
    int64_t lo, hi;
    cta_subslice(c, t, lo, hi);
    if (P.local_copy) ag_local_copy<U>(c, lo, hi);
    cta_signal_local(c, recdbl_partner(c.gi, 0), t);
  }
  char *my = P.recv[c.r];
  for (int k = 0; k < L; ++k) {
    const int partner = recdbl_partner(c.gi, k);
    const char *pr = P.recv[c.world(partner)];
    const int start = (partner >> k) << k, width = 1 << k;
    for (int t = 0; t < nsub; ++t) {
      if (!cta_wait(c, partner, k * nsub + t)) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int i = start; i < start + width; ++i)
        for (int j = 0; j < P.nsubblk; ++j)
          copy_units<U, kUnroll>(ag_block<U>(P, my, c.y, i, j), ag_block<U>(P, const_cast<char *>(pr), c.y, i, j), lo,
                                 hi);
      if (k + 1 < L) cta_signal_local(c, recdbl_partner(c.gi, k + 1), (k + 1) * nsub + t);
    }
  }
  cta_exit(c, partners, partners);
}


// ============================================================================
// direct all-gather data-movement variants (P.variant):
//   0 LDG pull (k_ag_direct), 1 STG push, 2 TMA pull, 3 TMA push.
// Push variants write into the peers' (symmetric) recv: the entry handshake
// means "my recv may be overwritten", the second one "my block has landed".
// ============================================================================
// dst2 != nullptr: the same loads are also stored to dst2 (my own output),
// so a push all-gather needs no separate local-copy pass.
template <int U>
__device__ __forceinline__ void store_units(char *dst, const char *src, int64_t lo, int64_t hi, char *dst2 = nullptr) {
  using T = typename VecT<U>::T;
  T *d = reinterpret_cast<T *>(dst);
  T *d2 = reinterpret_cast<T *>(dst2);
  const T *s = reinterpret_cast<const T *>(src);
  const int nt = blockDim.x;
  int64_t i = lo + threadIdx.x;
  for (; i + (int64_t)(kUnroll - 1) * nt < hi; i += (int64_t)kUnroll * nt) {
    T v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = __ldg(s + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) d[i + (int64_t)u * nt] = v[u];
    if (d2) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) d2[i + (int64_t)u * nt] = v[u];
    }
  }
  for (; i < hi; i += nt) {
    const T v = __ldg(s + i);
    d[i] = v;
    if (d2) d2[i] = v;
  }
}

template <int U>
__global__ void __launch_bounds__(kThreads) k_ag_direct_push(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const uint32_t peers = ((1u << c.gs) - 1) & ~(1u << c.gi);
  cta_signal_entry(c, peers);  // my recv may be written
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  if (P.item <= 0) {
    // Static slices, shift pattern: at step i every CTA of rank gi stores into
    // peer gi + i (each GPU sends to one peer and receives from one at a
    // time; a per-CTA rotation that spreads every GPU over all peers at once
    // measured 1-3 % slower). Each peer is waited for just before the first
    // store into it, not all of them up front.
    // The local copy of my block rides on the first peer's loads (one read of
    // send, two stores) instead of a separate pass in the kernel's tail.
    for (int i = 1; i < c.gs; ++i) {
      const int q = (c.gi + i) % c.gs;
      if (!cta_wait(c, q, 0)) return;
      char *dst = P.recv[c.world(q)];
      for (int t = 0; t < P.nsubblk; ++t)
        store_units<U>(ag_block<U>(P, dst, c.y, c.gi, t), P.send[c.r] + (int64_t)t * P.send_sub_stride * U, lo, hi,
                       (i == 1 && P.local_copy) ? ag_block<U>(P, P.recv[c.r], c.y, c.gi, t) : nullptr);
    }
    // Final publish: rank-level (one system release per rank) for flat calls;
    // per CTA in hierarchical phases, where a chained second launch's CTA b
    // starts as soon as this CTA b is done.
    if (P.rank_final) {
      cta_signal_rank(c, peers, 1);
    } else {
      cta_signal_mask(c, peers, 1);
    }
    if (P.local_copy && c.gs < 2) ag_local_copy<U>(c, lo, hi);
    if (!cta_wait_mask(c, peers, 1, P.rank_final ? 0 : -1)) return;
    return;
  }
  if (!cta_wait_mask(c, peers, 0)) return;
  {
    // items (range j, sub-block t, destination i), destination fastest
    const int nd = c.gs - 1;
    const int64_t nj = (P.blk + P.item - 1) / P.item;
    for_items(c, nj * nd * P.nsubblk, [&](int64_t id) {
      const int64_t j = id / (nd * P.nsubblk);
      const int rem = (int)(id - j * nd * P.nsubblk);
      const int q = (c.gi + 1 + rem % nd) % c.gs, t = rem / nd;
      const int64_t a = j * P.item, e = min(a + P.item, P.blk);
      store_units<U>(ag_block<U>(P, P.recv[c.world(q)], c.y, c.gi, t), P.send[c.r] + (int64_t)t * P.send_sub_stride * U,
                     a, e);
    });
  }
  if (P.rank_final) {
    cta_signal_rank(c, peers, 1);  // my whole block has landed in your recv (one system release per rank)
  } else {
    cta_signal_mask(c, peers, 1);
  }
  if (P.local_copy) ag_local_copy<U>(c, lo, hi);  // overlaps the peers' stores in flight
  if (!cta_wait_mask(c, peers, 1, P.rank_final ? 0 : -1)) return;
}

struct TmaCfg {
  static constexpr int kMaxStages = 8;
};

__device__ __forceinline__ TmaRing tma_ring_setup(char *dsm, int S, uint32_t T) {
  TmaRing R;
  R.buf = dsm;
  R.full = reinterpret_cast<uint64_t *>(dsm + (size_t)S * T);
  R.S = S;
  R.T = T;
  R.n = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(R.full + i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  return R;
}

template <bool PUSH>
__global__ void __launch_bounds__(kThreads) k_ag_direct_tma(const __grid_constant__ LaunchParams P) {
  extern __shared__ __align__(128) char dsm[];
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const uint32_t peers = ((1u << c.gs) - 1) & ~(1u << c.gi);
  TmaRing R = tma_ring_setup(dsm, P.tma_stages, P.tma_tile);
  cta_signal_mask(c, peers, 0);
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  if (!cta_wait_mask(c, peers, 0)) return;
  if (threadIdx.x == 0) {
    fence_proxy_async();
    const int gs = c.gs, nsb = P.nsubblk;
    const int nseg = gs * nsb;  // segment 0..nsb-1: own block (local copy)
    tma_copy_segments(R, nseg, [&](int i, char *&d, const char *&s, int64_t &len) {
      const int k = i / nsb, t = i % nsb;
      const int q = (c.gi + k) % gs;
      len = (hi - lo) * 16;
      if (k == 0) {
        if (!P.local_copy) { len = 0; d = nullptr; s = nullptr; return; }
        d = ag_block<16>(P, P.recv[c.r], c.y, c.gi, t) + lo * 16;
        s = P.send[c.r] + ((int64_t)t * P.send_sub_stride + lo) * 16;
      } else if (PUSH) {
        d = ag_block<16>(P, P.recv[c.world(q)], c.y, c.gi, t) + lo * 16;
        s = P.send[c.r] + ((int64_t)t * P.send_sub_stride + lo) * 16;
      } else {
        d = ag_block<16>(P, P.recv[c.r], c.y, q, t) + lo * 16;
        s = P.send[c.world(q)] + ((int64_t)t * P.send_sub_stride + lo) * 16;
      }
    });
  }
  if (PUSH) {
    cta_signal_mask(c, peers, 1);
    if (!cta_wait_mask(c, peers, 1)) return;
  } else {
    cta_exit(c, peers, peers);
  }
}

// ============================================================================
// reduce-scatter
// ============================================================================
// Chunk c (the part owned by member c) consists of nsubblk sub-blocks at
// (base + c*istride + t*sub_stride) units in send/work; the final chunk goes to
// out + t*out_sub_stride units.
template <typename T>
__device__ __forceinline__ char *rs_chunk(const LaunchParams &P, char *buf, int y, int c, int t) {
  return buf + (P.base[y] + (int64_t)c * P.istride + (int64_t)t * P.sub_stride) * (int64_t)sizeof(T);
}

template <int DT, bool VEC>
__global__ void __launch_bounds__(kThreads) k_rs_ring(const __grid_constant__ LaunchParams P) {
  using T = typename RUnit<DT, VEC>::T;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub;
  const int prev = ring_prev(c.gi, gs), next = ring_next(c.gi, gs);
  cta_signal_entry(c, 1u << next, nsub - 1);  // my send is ready (units 0..nsub-1)
  char *sendp = P.send[c.r], *workp = P.work[c.r], *outp = P.out[c.r];
  const int pw = c.world(prev);
  for (int s = 1; s < gs; ++s) {
    const int ch = ((c.gi - s - 1) % gs + gs) % gs;  // chunk whose carry I extend
    const bool last = (s == gs - 1);
    const char *remote = (s == 1) ? P.send[pw] : P.work[pw];
    for (int t = 0; t < nsub; ++t) {
      if (!cta_wait(c, prev, (s - 1) * nsub + t)) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int j = 0; j < P.nsubblk; ++j) {
        char *dst = last ? outp + (int64_t)j * P.out_sub_stride * (int64_t)sizeof(T) : rs_chunk<T>(P, workp, c.y, ch, j);
        reduce2_units<DT, VEC, kUnroll>(dst, rs_chunk<T>(P, sendp, c.y, ch, j),
                                        rs_chunk<T>(P, const_cast<char *>(remote), c.y, ch, j), lo, hi);
      }
      if (!last) cta_signal_local(c, next, s * nsub + t);
    }
  }
  cta_exit(c, 1u << prev, 1u << next);
}

template <int DT, bool VEC>
__global__ void __launch_bounds__(kThreads) k_rs_rec(const __grid_constant__ LaunchParams P) {
  using T = typename RUnit<DT, VEC>::T;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub, L = ilog2(gs);
  uint32_t partners = 0;
  for (int k = 0; k < L; ++k) partners |= 1u << rechalf_partner(c.gi, gs, k);
  cta_signal_entry(c, 1u << rechalf_partner(c.gi, gs, 0), nsub - 1);  // my send is ready (units 0..nsub-1)
  char *sendp = P.send[c.r], *workp = P.work[c.r], *outp = P.out[c.r];
  int lo_c = 0, hi_c = gs;
  for (int k = 0; k < L; ++k) {
    const int half = (hi_c - lo_c) / 2, mid = lo_c + half;
    const int partner = c.gi ^ half;  // == rechalf_partner(c.gi, gs, k)
    int m0, m1;
    if (c.gi < mid) { m0 = lo_c; m1 = mid; } else { m0 = mid; m1 = hi_c; }
    const bool last = (k == L - 1);
    const int pw = c.world(partner);
    const char *remote = (k == 0) ? P.send[pw] : P.work[pw];
    const char *local = (k == 0) ? sendp : workp;
    for (int t = 0; t < nsub; ++t) {
      if (!cta_wait(c, partner, k * nsub + t)) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int ch = m0; ch < m1; ++ch)
        for (int j = 0; j < P.nsubblk; ++j) {
          char *dst = last ? outp + (int64_t)j * P.out_sub_stride * (int64_t)sizeof(T) : rs_chunk<T>(P, workp, c.y, ch, j);
          reduce2_units<DT, VEC, kUnroll>(dst, rs_chunk<T>(P, const_cast<char *>(local), c.y, ch, j),
                                          rs_chunk<T>(P, const_cast<char *>(remote), c.y, ch, j), lo, hi);
        }
      if (!last) cta_signal_local(c, rechalf_partner(c.gi, gs, k + 1), (k + 1) * nsub + t);
    }
    lo_c = m0;
    hi_c = m1;
  }
  cta_exit(c, partners, partners);
}


// RS recursive halving, pull, with per-step dynamic work items (rs_variant 7).
// The static kernel above ties slice b to CTA b in every step, so a CTA whose
// partner CTA was slow in step k waits at the boundary and the last CTAs form
// a tail (profiles/r2_overhead_p4.md: boundary 3-5 us, tail 8 us at p=4).
// Here every step's element range is cut into P.item-unit items claimed from
// a per-step counter (CTRL[3 + k]); item i of step k waits for item i of
// step k-1 on this rank (F_ITEM[gi][i], local) and on the partner
// (F_ITEM[partner][i], remote), and publishes its own completion to the next
// partner and to itself. Same arithmetic and order as k_rs_rec (butterfly,
// wire rounding per step): bit-identical results. Exit: every CTA b signals
// DONE to the partners and waits for theirs (a rank's kernel completes only
// after all its CTAs, so the union over b covers every item).
template <int DT, bool VEC>
__global__ void __launch_bounds__(kThreads) k_rs_rec_items(const __grid_constant__ LaunchParams P) {
  using T = typename RUnit<DT, VEC>::T;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, L = ilog2(gs);
  uint32_t partners = 0;
  for (int k = 0; k < L; ++k) partners |= 1u << rechalf_partner(c.gi, gs, k);
  const int p0 = rechalf_partner(c.gi, gs, 0);
  cta_signal_entry(c, 1u << p0, 0);  // my send is ready (read by partner_0 in step 0)
  if (!cta_wait(c, p0, 0)) return;    // partner_0's send is ready
  char *sendp = P.send[c.r], *workp = P.work[c.r], *outp = P.out[c.r];
  const int64_t I = P.item;
  const int64_t nitems = (P.blk + I - 1) / I;
  int lo_c = 0, hi_c = gs;
  bool ok = true;
  for (int k = 0; k < L && ok; ++k) {
    const int half = (hi_c - lo_c) / 2, mid = lo_c + half;
    const int partner = c.gi ^ half;
    int m0, m1;
    if (c.gi < mid) { m0 = lo_c; m1 = mid; } else { m0 = mid; m1 = hi_c; }
    const bool last = (k == L - 1);
    const int pw = c.world(partner);
    const char *remote = (k == 0) ? P.send[pw] : P.work[pw];
    const char *local = (k == 0) ? sendp : workp;
    const int next = last ? -1 : rechalf_partner(c.gi, gs, k + 1);
    for_items(c, nitems, [&](int64_t it) {
      if (!ok) return;
      if (k > 0 && (!item_wait(c, c.gi, (int)it, k) || !item_wait(c, partner, (int)it, k))) { ok = false; return; }
      const int64_t lo = it * I, hi = lo + I < P.blk ? lo + I : P.blk;
      for (int ch = m0; ch < m1; ++ch)
        for (int j = 0; j < P.nsubblk; ++j) {
          char *dst = last ? outp + (int64_t)j * P.out_sub_stride * (int64_t)sizeof(T) : rs_chunk<T>(P, workp, c.y, ch, j);
          reduce2_units<DT, VEC, kUnroll>(dst, rs_chunk<T>(P, const_cast<char *>(local), c.y, ch, j),
                                          rs_chunk<T>(P, const_cast<char *>(remote), c.y, ch, j), lo, hi);
        }
      if (!last) item_signal(c, next, (int)it, k + 1);
    }, 3 + k);
    lo_c = m0;
    hi_c = m1;
  }
  if (!ok) return;
  cta_exit(c, partners, partners);
}

// ============================================================================
// PUSH family (ag_variant / rs_variant 1). Data moves as posted NVLink stores
// into the consumer's symmetric buffer; the consumer only reads local HBM.
// Channel protocol per (writer -> reader) pair: unit 0 travels reader ->
// writer ("my receive buffer is free": the reader's kernel for this call has
// started, so nothing of the previous call still reads it), data units
// 1 + step*nsub + t travel writer -> reader after the stores of that
// sub-slice (release after a CTA barrier). No exit barrier is needed: a
// writer only reads its own buffers.
// ============================================================================
__device__ __forceinline__ int push_unit(int step, int nsub, int t) { return 1 + step * nsub + t; }

// AG ring, push: step s forwards block (gi - s) to next's recv.
template <int U>
__global__ void __launch_bounds__(kThreads) k_ag_ring_push(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub;
  const int prev = ring_prev(c.gi, gs), next = ring_next(c.gi, gs);
  cta_signal_entry(c, 1u << prev);  // my recv is free
  if (!cta_wait(c, next, 0)) return;
  char *my = P.recv[c.r];
  char *nx = P.recv[c.world(next)];
  for (int s = 0; s < gs - 1; ++s) {
    const int blk = (c.gi - s + gs) % gs;
    for (int t = 0; t < nsub; ++t) {
      if (s > 0 && !cta_wait(c, prev, push_unit(s - 1, nsub, t))) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int j = 0; j < P.nsubblk; ++j) {
        // my own block comes from send (and is stored into my recv by the
        // same loads), or is already in place in recv (local_copy == 0)
        if (s == 0 && P.local_copy)
          copy_units_dup<U, kUnroll>(ag_block<U>(P, nx, c.y, blk, j), ag_block<U>(P, my, c.y, blk, j),
                                     P.send[c.r] + (int64_t)j * P.send_sub_stride * U, lo, hi);
        else
          copy_units<U, kUnroll>(ag_block<U>(P, nx, c.y, blk, j), ag_block<U>(P, my, c.y, blk, j), lo, hi);
      }
      if (s == gs - 2 && nsub == 1 && P.rank_final)
        cta_signal_rank(c, 1u << next, push_unit(s, nsub, t));  // final unit: one system release per rank
      else
        cta_signal(c, next, push_unit(s, nsub, t));
    }
  }
  if (gs > 1 && nsub == 1 && P.rank_final) {
    if (!cta_wait_mask(c, 1u << prev, push_unit(gs - 2, 1, 0), 0)) return;
  } else {
    for (int t = 0; t < nsub; ++t)
      if (!cta_wait(c, prev, push_unit(gs - 2, nsub, t))) return;
  }
  if (P.local_copy && gs < 2) {
    int64_t lo, hi;
    split32(P.blk, P.ctas, c.b, lo, hi);
    ag_local_copy<U>(c, lo, hi);
  }
}

// AG recursive doubling, push: step k sends my 2^k gathered blocks to r ^ 2^k.
template <int U>
__global__ void __launch_bounds__(kThreads) k_ag_rec_push(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub, L = ilog2(gs);
  uint32_t partners = 0;
  for (int k = 0; k < L; ++k) partners |= 1u << recdbl_partner(c.gi, k);
  cta_signal_entry(c, partners);  // my recv is free
  char *my = P.recv[c.r];
  for (int k = 0; k < L; ++k) {
    const int partner = recdbl_partner(c.gi, k);
    if (!cta_wait(c, partner, 0)) return;
    char *pr = P.recv[c.world(partner)];
    const int start = (c.gi >> k) << k, width = 1 << k;
    for (int t = 0; t < nsub; ++t) {
      if (k > 0 && !cta_wait(c, recdbl_partner(c.gi, k - 1), push_unit(k - 1, nsub, t))) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int i = start; i < start + width; ++i)
        for (int j = 0; j < P.nsubblk; ++j) {
          // my own block comes from send; at step 0 the same loads also
          // store it into my recv (no local-copy pass in the tail)
          const char *mine = P.send[c.r] + (int64_t)j * P.send_sub_stride * U;
          if (i == c.gi && P.local_copy && k == 0)
            copy_units_dup<U, kUnroll>(ag_block<U>(P, pr, c.y, i, j), ag_block<U>(P, my, c.y, i, j), mine, lo, hi);
          else if (i == c.gi && P.local_copy)
            copy_units<U, kUnroll>(ag_block<U>(P, pr, c.y, i, j), mine, lo, hi);
          else
            copy_units<U, kUnroll>(ag_block<U>(P, pr, c.y, i, j), ag_block<U>(P, my, c.y, i, j), lo, hi);
        }
      if (k == L - 1 && nsub == 1 && P.rank_final)
        cta_signal_rank(c, 1u << partner, push_unit(k, nsub, t));  // final unit: one system release per rank
      else
        cta_signal(c, partner, push_unit(k, nsub, t));
    }
  }
  if (L > 0 && nsub == 1 && P.rank_final) {
    if (!cta_wait_mask(c, 1u << recdbl_partner(c.gi, L - 1), push_unit(L - 1, 1, 0), 0)) return;
  } else {
    for (int t = 0; t < nsub; ++t)
      if (!cta_wait(c, recdbl_partner(c.gi, L - 1), push_unit(L - 1, nsub, t))) return;
  }
  if (P.local_copy && L == 0) {
    int64_t lo, hi;
    split32(P.blk, P.ctas, c.b, lo, hi);
    ag_local_copy<U>(c, lo, hi);
  }
}

// RS ring, push with the add at the sender: v = own chunk + carry received in
// my staging, stored into next's staging (or my output on the last step).
template <int DT, bool VEC>
__global__ void __launch_bounds__(kThreads) k_rs_ring_push(const __grid_constant__ LaunchParams P) {
  using T = typename RUnit<DT, VEC>::T;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub;
  const int prev = ring_prev(c.gi, gs), next = ring_next(c.gi, gs);
  cta_signal_entry(c, 1u << prev);  // my staging is free
  if (!cta_wait(c, next, 0)) return;
  char *sendp = P.send[c.r], *stg = P.recv[c.r], *nstg = P.recv[c.world(next)], *outp = P.out[c.r];
  {
    const int ch = (c.gi - 1 + gs) % gs;  // initial carry (collectives.py:98)
    for (int t = 0; t < nsub; ++t) {
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int j = 0; j < P.nsubblk; ++j)
        copy_units<(int)sizeof(T), kUnroll>(rs_chunk<T>(P, nstg, c.y, ch, j), rs_chunk<T>(P, sendp, c.y, ch, j), lo, hi);
      cta_signal(c, next, push_unit(0, nsub, t));
    }
  }
  for (int s = 1; s < gs; ++s) {
    const int ch = ((c.gi - s - 1) % gs + gs) % gs;
    const bool last = (s == gs - 1);
    for (int t = 0; t < nsub; ++t) {
      if (!cta_wait(c, prev, push_unit(s - 1, nsub, t))) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int j = 0; j < P.nsubblk; ++j) {
        char *dst = last ? outp + (int64_t)j * P.out_sub_stride * (int64_t)sizeof(T) : rs_chunk<T>(P, nstg, c.y, ch, j);
        reduce2_units<DT, VEC, kUnroll>(dst, rs_chunk<T>(P, sendp, c.y, ch, j), rs_chunk<T>(P, stg, c.y, ch, j), lo, hi);
      }
      if (!last) cta_signal(c, next, push_unit(s, nsub, t));
    }
  }
}

// RS recursive halving, push with the add at the sender. Staging region k
// (chunks [gs - gs/2^k, ...)) receives partner_k's partial over mine_k; the
// result of step k is written locally for mine_{k+1} and straight into
// partner_{k+1}'s staging region k+1 for theirs_{k+1}.
template <int DT, bool VEC>
__global__ void __launch_bounds__(kThreads) k_rs_rec_push(const __grid_constant__ LaunchParams P) {
  using T = typename RUnit<DT, VEC>::T;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, nsub = P.nsub, L = ilog2(gs);
  uint32_t partners = 0;
  for (int k = 0; k < L; ++k) partners |= 1u << rechalf_partner(c.gi, gs, k);
  cta_signal_entry(c, partners);  // my staging is free
  char *sendp = P.send[c.r], *workp = P.work[c.r], *outp = P.out[c.r], *stgp = P.recv[c.r];
  // staging slot of absolute chunk ch received at step k (region base = gs - gs/2^k chunks)
  auto stg_chunk = [&](char *buf, int k, int lo_k, int ch, int j) -> char * {
    const int slot = (gs - (gs >> k)) + (ch - lo_k);
    return rs_chunk<T>(P, buf, c.y, slot, j);
  };
  // step "-1": raw input over theirs_0 into partner_0's staging region 0
  {
    const int partner = rechalf_partner(c.gi, gs, 0);
    if (!cta_wait(c, partner, 0)) return;
    const int half = gs / 2, mid = half;
    const int t0 = c.gi < mid ? mid : 0, t1 = c.gi < mid ? gs : mid;  // theirs_0
    char *pst = P.recv[c.world(partner)];
    for (int t = 0; t < nsub; ++t) {
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int ch = t0; ch < t1; ++ch)
        for (int j = 0; j < P.nsubblk; ++j)
          copy_units<(int)sizeof(T), kUnroll>(stg_chunk(pst, 0, t0, ch, j), rs_chunk<T>(P, sendp, c.y, ch, j), lo, hi);
      cta_signal(c, partner, push_unit(0, nsub, t));
    }
  }
  int lo_c = 0, hi_c = gs;
  for (int k = 0; k < L; ++k) {
    const int half = (hi_c - lo_c) / 2, mid = lo_c + half;
    const int partner = c.gi ^ half;  // == rechalf_partner(c.gi, gs, k)
    int m0, m1;
    if (c.gi < mid) { m0 = lo_c; m1 = mid; } else { m0 = mid; m1 = hi_c; }
    const bool last = (k == L - 1);
    // next step's split of mine_k
    int n0 = m0, n1 = m1, nxt = -1;
    char *nst = nullptr;
    if (!last) {
      const int h2 = (m1 - m0) / 2, mid2 = m0 + h2;
      if (c.gi < mid2) { n0 = m0; n1 = mid2; } else { n0 = mid2; n1 = m1; }
      nxt = c.gi ^ h2;
      if (!cta_wait(c, nxt, 0)) return;
      nst = P.recv[c.world(nxt)];
    }
    const int t_lo = (n0 == m0) ? n1 : m0;  // theirs_{k+1} = mine_k \ mine_{k+1}
    const char *local = (k == 0) ? sendp : workp;
    for (int t = 0; t < nsub; ++t) {
      if (!cta_wait(c, partner, push_unit(k, nsub, t))) return;
      int64_t lo, hi;
      cta_subslice(c, t, lo, hi);
      for (int ch = m0; ch < m1; ++ch)
        for (int j = 0; j < P.nsubblk; ++j) {
          char *dst;
          if (last) dst = outp + (int64_t)j * P.out_sub_stride * (int64_t)sizeof(T);
          else if (ch >= n0 && ch < n1) dst = rs_chunk<T>(P, workp, c.y, ch, j);
          else dst = stg_chunk(nst, k + 1, t_lo, ch, j);
          reduce2_units<DT, VEC, kUnroll>(dst, rs_chunk<T>(P, const_cast<char *>(local), c.y, ch, j),
                                          stg_chunk(stgp, k, m0, ch, j), lo, hi);
        }
      if (!last) cta_signal(c, nxt, push_unit(k + 1, nsub, t));
    }
    lo_c = m0;
    hi_c = m1;
  }
}

// Direct reduce-scatter, one step. PULL: every member's chunk `gi` is read
// from the peers' symmetric send buffers. PUSH: every rank first stores its
// chunk q into member q's staging slot [gi] (posted NVLink writes), then folds
// its own slots locally. Either way the leaves are loaded first (MAXP
// independent 16-byte loads in flight per thread) and combined with static
// register indices in the named order.
template <typename T>
__device__ __forceinline__ void copy_typed(T *d, const T *s, int64_t lo, int64_t hi) {
  const int nt = blockDim.x;
  int64_t i = lo + threadIdx.x;
  for (; i + (int64_t)(kUnroll - 1) * nt < hi; i += (int64_t)kUnroll * nt) {
    T v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = __ldg(s + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) d[i + (int64_t)u * nt] = v[u];
  }
  for (; i < hi; i += nt) d[i] = __ldg(s + i);
}

// Fold the MAXP leaves src[i][off + e] of every element e in [lo, hi) in the
// named order (registers only, fp32 accumulation) and store to dst[e].
// wire = true: the partial is rounded to the storage type after every add, as
// the step-wise kernels store it between steps (bit-identical to ring /
// recursive halving in bf16 / fp16; a no-op for fp32).
template <int DT, bool VEC, int ORDER, int MAXP>
__device__ __forceinline__ void rs_fold(const typename RUnit<DT, VEC>::T *const *src, int gs, int64_t off,
                                        typename RUnit<DT, VEC>::T *dst, int64_t lo, int64_t hi, bool wire = false) {
  using R = RUnit<DT, VEC>;
  using T = typename R::T;
  using Acc = typename R::Acc;
  const int nt = blockDim.x;
  // EU elements per thread per iteration keep >= 8 independent 16-byte
  // loads in flight also for small groups (p = 2: 2 leaves per element)
  constexpr int EU = MAXP >= 8 ? 1 : 8 / MAXP;
  for (int64_t e0 = lo + threadIdx.x; e0 < hi; e0 += (int64_t)EU * nt) {
    T rawu[EU][MAXP];
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      const int64_t e = e0 + (int64_t)u * nt;
#pragma unroll
      for (int i = 0; i < MAXP; ++i) rawu[u][i] = (i < gs && e < hi) ? ld_peer(src[i] + off + e) : T{};
    }
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      const int64_t e = e0 + (int64_t)u * nt;
      if (e >= hi) break;
      const T *raw = rawu[u];
      Acc acc;
      if (ORDER == O_REC) {
        Acc v[MAXP];
#pragma unroll
        for (int i = 0; i < MAXP; ++i) v[i] = R::load(raw[i]);
#pragma unroll
        for (int h = MAXP / 2; h >= 1; h >>= 1) {
          if (h < gs) {  // levels above the group size do not exist (gs <= MAXP)
#pragma unroll
            for (int m = 0; m < h; ++m) {
              acc_add<Acc, R::N>(v[m], v[m ^ h]);
              if (DT != DT_F32 && wire) v[m] = R::load(R::store(v[m]));
            }
          }
        }
        acc = v[0];
      } else if (ORDER == O_RANK) {
#pragma unroll
        for (int k = 0; k < R::N; ++k) acc.v[k] = 0.0f;
#pragma unroll
        for (int i = 0; i < MAXP; ++i)
          if (i < gs) acc_add<Acc, R::N>(acc, R::load(raw[i]));
      } else {
        acc = R::load(raw[0]);
#pragma unroll
        for (int i = 1; i < MAXP; ++i)
          if (i < gs) {
            acc_add<Acc, R::N>(acc, R::load(raw[i]));
            if (DT != DT_F32 && wire) acc = R::load(R::store(acc));
          }
      }
      dst[e] = R::store(acc);
    }
  }
}

template <int DT, bool VEC, int ORDER, int MAXP, bool PUSH>
__global__ void __launch_bounds__(kThreads) k_rs_direct(const __grid_constant__ LaunchParams P) {
  using R = RUnit<DT, VEC>;
  using T = typename R::T;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, gi = c.gi;
  const uint32_t peers = ((1u << gs) - 1) & ~(1u << gi);
  cta_signal_entry(c, peers);  // pull: my send is ready; push: my staging is free
  if (!cta_wait_mask(c, peers, 0)) return;
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  const T *own = reinterpret_cast<const T *>(P.send[c.r]);
  if (PUSH) {
    // Static slices only: the fold below consumes, inside this launch, exactly
    // the slice that the peers' CTA b pushed and signalled to my CTA b, so
    // the push may not be redistributed by work items (P.item is ignored).
    for (int i = 1; i < gs; ++i) {
      const int q = (gi + i) % gs;
      T *dst = reinterpret_cast<T *>(P.recv[c.world(q)]) + (int64_t)gi * P.blk;
      copy_typed<T>(dst, own + P.base[c.y] + (int64_t)q * P.istride, lo, hi);
    }
    cta_signal_mask(c, peers, 1);  // my chunks have landed
    if (!cta_wait_mask(c, peers, 1)) return;
  }
  const T *src[MAXP];
#pragma unroll
  for (int i = 0; i < MAXP; ++i) {
    int q;
    if (ORDER == O_RING) q = (gi + 1 + i) % gs;
    else if (ORDER == O_REC) q = gi ^ i;
    else q = i;
    if (i >= gs) q = gi;
    if (PUSH)
      src[i] = (q == gi) ? own + P.base[c.y] + (int64_t)gi * P.istride
                         : reinterpret_cast<const T *>(P.recv[c.r]) + (int64_t)q * P.blk;
    else
      src[i] = reinterpret_cast<const T *>(P.send[c.world(q)]) + P.base[c.y] + (int64_t)gi * P.istride;
  }
  auto fold = [&](int j, int64_t lo, int64_t hi) {
    rs_fold<DT, VEC, ORDER, MAXP>(src, gs, (int64_t)j * P.sub_stride,
                                  reinterpret_cast<T *>(P.out[c.r]) + (int64_t)j * P.out_sub_stride, lo, hi,
                                  P.wire != 0);
  };
  if (!PUSH && P.item > 0) {  // pull: items (range, sub-block)
    const int64_t nj = (P.blk + P.item - 1) / P.item;
    for_items(c, nj * P.nsubblk, [&](int64_t id) {
      const int64_t j = id / P.nsubblk;
      const int64_t a = j * P.item;
      fold((int)(id - j * P.nsubblk), a, min(a + P.item, P.blk));
    });
  } else {
    for (int j = 0; j < P.nsubblk; ++j) fold(j, lo, hi);
  }
  if (!PUSH) cta_exit(c, peers, peers);
}


// Direct reduce-scatter, pipelined push (rs_variant 5). CTAs [0, C) push,
// CTAs [C, 2C) fold: pusher b stores sub-slice t of every chunk q into
// member q's staging slot [gi] and publishes unit t+1 to q in the READY
// words of CTA index b; folder C+b waits for unit t+1 from every peer's
// pusher b and folds sub-slice t from local memory, so the fold of t runs
// while the pushes of t+1.. are in flight (NVLink and HBM busy at once) and
// the data travels as posted writes (all-to-all: 668-682 GB/s vs 628-637 for
// peer loads, profiles/r1_engine_probe_p4.md). Entry: every pusher b
// announces "my staging is free" to the peers' pushers b. No exit barrier:
// folders read only local memory.
template <int DT, bool VEC, int ORDER, int MAXP>
__global__ void __launch_bounds__(kThreads) k_rs_direct_pp(const __grid_constant__ LaunchParams P) {
  using R = RUnit<DT, VEC>;
  using T = typename R::T;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const int gs = c.gs, gi = c.gi, C = P.ctas / 2, nsub = P.nsub > 1 ? P.nsub : 4;
  const uint32_t peers = ((1u << gs) - 1) & ~(1u << gi);
  const bool pusher = c.b < C;
  const int b = pusher ? c.b : c.b - C;
  if (b >= C) return;  // odd grid: the spare CTA has no slice
  int64_t lo, hi;
  split32(P.blk, C, b, lo, hi);
  const T *own = reinterpret_cast<const T *>(P.send[c.r]) + P.base[c.y];
  if (pusher) {
    cta_signal_entry(c, peers);  // my staging is free
    if (!cta_wait_mask(c, peers, 0)) return;
    for (int t = 0; t < nsub; ++t) {
      int64_t a, e;
      split32(hi - lo, nsub, t, a, e);
      for (int i = 1; i < gs; ++i) {
        const int q = (gi + i) % gs;
        copy_typed<T>(reinterpret_cast<T *>(P.recv[c.world(q)]) + (int64_t)gi * P.blk, own + (int64_t)q * P.istride,
                      lo + a, lo + e);
      }
      cta_signal_mask(c, peers, t + 1);  // sub-slice t of my chunks has landed
    }
    return;
  }
  const T *src[MAXP];
#pragma unroll
  for (int i = 0; i < MAXP; ++i) {
    int q;
    if (ORDER == O_RING) q = (gi + 1 + i) % gs;
    else if (ORDER == O_REC) q = gi ^ i;
    else q = i;
    if (i >= gs) q = gi;
    src[i] = (q == gi) ? own + (int64_t)gi * P.istride : reinterpret_cast<const T *>(P.recv[c.r]) + (int64_t)q * P.blk;
  }
  T *dst = reinterpret_cast<T *>(P.out[c.r]);
  for (int t = 0; t < nsub; ++t) {
    if (!cta_wait_mask(c, peers, t + 1, b)) return;
    int64_t a, e;
    split32(hi - lo, nsub, t, a, e);
    rs_fold<DT, VEC, ORDER, MAXP>(src, gs, 0, dst, lo + a, lo + e, P.wire != 0);
  }
}

// ============================================================================
// LL direct collectives (small messages; protocol in device.cuh)
// ============================================================================
// Payload unit = 8 bytes (P.blk etc. are in 8-byte units). Every CTA owns
// units [lo,hi) of each (sub-)block: it posts them to every peer, then reads
// the peers' words of the same range — all peers' loads issued before any is
// waited on — and writes them out locally.
template <int MAXP>
__global__ void __launch_bounds__(kThreads) k_ag_direct_ll(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  __shared__ uint32_t s_tag[PCCL_MAXR];
  ll_tags(c, s_tag);
  const int gs = c.gs, gi = c.gi, nt = blockDim.x;
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  ll_post_headers(c, s_tag);
  for (int t = 0; t < P.nsubblk; ++t) {
    const uint2 *src = reinterpret_cast<const uint2 *>(P.send[c.r]) + (int64_t)t * P.send_sub_stride;
    uint2 *mine = reinterpret_cast<uint2 *>(ag_block<8>(P, P.recv[c.r], c.y, gi, t));
    for (int64_t e = lo + threadIdx.x; e < hi; e += nt) {
      const uint2 v = __ldg(src + e);
#pragma unroll
      for (int i = 1; i < MAXP; ++i) {
        if (i >= gs) break;
        const int q = (gi + i) % gs;
        uint4 *d = reinterpret_cast<uint4 *>(ll_region(P, c.world(q), s_tag[q], c.r) + PCCL_LL_HDR_BYTES);
        ll_st(d + (int64_t)t * P.blk + e, v.x, v.y, s_tag[q]);
      }
      if (P.local_copy) mine[e] = v;
    }
  }
  int code = 0;
  for (int t = 0; t < P.nsubblk && !code; ++t) {
    for (int64_t e = lo + threadIdx.x; e < hi && !code; e += nt) {
      uint4 v[MAXP];
#pragma unroll
      for (int i = 1; i < MAXP; ++i) {
        if (i < gs) {
          const int q = (gi + gs - i) % gs;
          v[i] = ll_ld(reinterpret_cast<const uint4 *>(ll_region(P, c.r, s_tag[q], c.world(q)) + PCCL_LL_HDR_BYTES) +
                       (int64_t)t * P.blk + e);
        }
      }
#pragma unroll
      for (int i = 1; i < MAXP; ++i) {
        if (i < gs && !code) {
          const int q = (gi + gs - i) % gs;
          const char *reg = ll_region(P, c.r, s_tag[q], c.world(q));
          if (!ll_ok(v[i], s_tag[q]))
            code = ll_wait(c, reinterpret_cast<const uint4 *>(reg + PCCL_LL_HDR_BYTES) + (int64_t)t * P.blk + e,
                           s_tag[q], v[i], reinterpret_cast<const uint4 *>(reg));
          reinterpret_cast<uint2 *>(ag_block<8>(P, P.recv[c.r], c.y, q, t))[e] = make_uint2(v[i].x, v[i].z);
        }
      }
    }
  }
  ll_finish(c, s_tag, code);
}

// 8 payload bytes as N accumulator lanes
template <int DT> struct LLU;
template <> struct LLU<DT_F32> {
  static constexpr int N = 2;
  struct Acc { float v[2]; };
  static __device__ __forceinline__ Acc load(uint2 u) { Acc a; a.v[0] = __uint_as_float(u.x); a.v[1] = __uint_as_float(u.y); return a; }
  static __device__ __forceinline__ uint2 store(const Acc &a) { return make_uint2(__float_as_uint(a.v[0]), __float_as_uint(a.v[1])); }
};
template <> struct LLU<DT_BF16> {
  static constexpr int N = 4;
  struct Acc { float v[4]; };
  static __device__ __forceinline__ Acc load(uint2 u) {
    Acc a; float2 f = bf2_to_f2(u.x); a.v[0] = f.x; a.v[1] = f.y; f = bf2_to_f2(u.y); a.v[2] = f.x; a.v[3] = f.y; return a;
  }
  static __device__ __forceinline__ uint2 store(const Acc &a) {
    return make_uint2(f2_to_bf2(a.v[0], a.v[1]), f2_to_bf2(a.v[2], a.v[3]));
  }
};
template <> struct LLU<DT_F16> {
  static constexpr int N = 4;
  struct Acc { float v[4]; };
  static __device__ __forceinline__ Acc load(uint2 u) {
    Acc a; float2 f = h2_to_f2(u.x); a.v[0] = f.x; a.v[1] = f.y; f = h2_to_f2(u.y); a.v[2] = f.x; a.v[3] = f.y; return a;
  }
  static __device__ __forceinline__ uint2 store(const Acc &a) {
    return make_uint2(f2_to_h2(a.v[0], a.v[1]), f2_to_h2(a.v[2], a.v[3]));
  }
};

// ============================================================================
// LL128: a line protocol for mid-size direct all-gathers. A 128-byte line is
// written by 8 lanes of ONE warp store instruction (16 bytes each): 120
// payload bytes and, in the last 8, the channel's message tag. A line is
// delivered over NVLink as a unit (tools/ll128_probe.cu: no torn line in
// 12.8 GB per direction), so a reader whose warp sees the tag in all four
// lines of its 512-byte load holds their payload: no handshake, no fence, no
// exit barrier, 94 % payload efficiency (LL: 50 %). Regions, channel
// counters and the signature header follow the LL protocol (see device.cuh),
// in a separate set of regions.
// ============================================================================
__device__ __forceinline__ void st_line16(uint64_t *p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_line16(const uint64_t *p, uint64_t &a, uint64_t &b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// slow path of a waiting warp (lane 0): world error, signature mismatch, timeout
__device__ __noinline__ int ll128_slow_check(const Ctx &c, const char *reg, uint32_t tag) {
  if (const uint64_t e = *err_mirror(*c.P, c.r)) return (int)e;
  const uint4 h = ll_ld(reinterpret_cast<const uint4 *>(reg));
  if (ll_ok(h, tag) && (h.x != c.P->meta[c.y] || h.z != c.P->meta[c.y])) return 4;
  if (global_timer_ns() - c.t0 > (uint64_t)c.P->timeout_ns) return 5;
  return 0;
}

template <int MAXP>
__global__ void __launch_bounds__(kThreads) k_ag_direct_ll128(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  c.ll_ctr = PCCL_WCTRL_LL128;
  CtaEpilogue fin(c);
  __shared__ uint32_t s_tag[PCCL_MAXR];
  ll_tags(c, s_tag);
  ll_post_headers(c, s_tag);
  const int gs = c.gs, gi = c.gi;
  const int lane = threadIdx.x & 31, j = lane & 7;
  const int64_t words = P.blk;  // 8-byte units of my block
  const int64_t lines = (words + 14) / 15;
  const int64_t nw = (int64_t)P.ctas * (blockDim.x >> 5);
  const int64_t w0 = (int64_t)c.b * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t *src = reinterpret_cast<const uint64_t *>(P.send[c.r]);
  uint64_t *mine = reinterpret_cast<uint64_t *>(ag_block<8>(P, P.recv[c.r], c.y, gi, 0));
  // send: each warp packs 4 lines (lane j of a line: words 2j, 2j+1; lane 7:
  // word 14 and the tag) and stores them into every peer's region
  for (int64_t g = w0; g * 4 < lines; g += nw) {
    const int64_t line = g * 4 + (lane >> 3);
    if (line >= lines) continue;
    const int64_t wa = line * 15 + 2 * j;
    uint64_t a = 0, b = 0;
    if (wa < words) a = src[wa];
    if (j < 7 && wa + 1 < words) b = src[wa + 1];
    if (P.local_copy) {
      if (wa < words) mine[wa] = a;
      if (j < 7 && wa + 1 < words) mine[wa + 1] = b;
    }
#pragma unroll
    for (int i = 1; i < MAXP; ++i) {
      if (i >= gs) break;
      const int q = (gi + i) % gs;
      uint64_t *d = reinterpret_cast<uint64_t *>(ll128_region(P, c.world(q), s_tag[q], c.r) + PCCL_LL_HDR_BYTES);
      st_line16(d + line * 16 + 2 * j, a, j < 7 ? b : (uint64_t)s_tag[q]);
    }
  }
  // receive: poll each source's lines until the warp sees the tag in all of
  // them, then scatter the payload into that source's block
  int code = 0;
  for (int i = 1; i < MAXP; ++i) {
    if (i >= gs || code) break;
    const int q = (gi + gs - i) % gs;
    const char *reg = ll128_region(P, c.r, s_tag[q], c.world(q));
    const uint64_t *base = reinterpret_cast<const uint64_t *>(reg + PCCL_LL_HDR_BYTES);
    uint64_t *out = reinterpret_cast<uint64_t *>(ag_block<8>(P, P.recv[c.r], c.y, q, 0));
    const uint64_t tag = s_tag[q];
    for (int64_t g = w0; g * 4 < lines; g += nw) {
      const int64_t line = g * 4 + (lane >> 3);
      const bool valid = line < lines;
      const uint64_t *pl = base + (valid ? line : 0) * 16 + 2 * j;
      uint64_t a, b;
      uint32_t it = 0;
      while (true) {
        ld_line16(pl, a, b);
        if (__all_sync(0xffffffffu, !valid || j != 7 || b == tag)) break;
        if ((++it & 1023u) == 0) {
          int e = lane == 0 ? ll128_slow_check(c, reg, (uint32_t)tag) : 0;
          e = __shfl_sync(0xffffffffu, e, 0);
          if (e) {
            code = e;
            break;
          }
        }
      }
      if (code) break;
      if (valid) {
        const int64_t wa = line * 15 + 2 * j;
        if (wa < words) out[wa] = a;
        if (j < 7 && wa + 1 < words) out[wa + 1] = b;
      }
    }
  }
  ll_finish(c, s_tag, code);
}

// Chunk q of my input goes to member q as an LL message; my output chunk is
// folded from my own chunk and the p-1 received ones in the named order
// (same folds as k_rs_direct, so results are bit-identical to it).
template <int DT, int ORDER, int MAXP>
__global__ void __launch_bounds__(kThreads) k_rs_direct_ll(const __grid_constant__ LaunchParams P) {
  using R = LLU<DT>;
  using Acc = typename R::Acc;
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  __shared__ uint32_t s_tag[PCCL_MAXR];
  ll_tags(c, s_tag);
  const int gs = c.gs, gi = c.gi, nt = blockDim.x;
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  const uint2 *own = reinterpret_cast<const uint2 *>(P.send[c.r]) + P.base[c.y];
  ll_post_headers(c, s_tag);
  for (int i = 1; i < gs; ++i) {
    const int q = (gi + i) % gs;
    uint4 *d = reinterpret_cast<uint4 *>(ll_region(P, c.world(q), s_tag[q], c.r) + PCCL_LL_HDR_BYTES);
    for (int j = 0; j < P.nsubblk; ++j) {
      const uint2 *src = own + (int64_t)q * P.istride + (int64_t)j * P.sub_stride;
      for (int64_t e = lo + threadIdx.x; e < hi; e += nt) {
        const uint2 v = __ldg(src + e);
        ll_st(d + (int64_t)j * P.blk + e, v.x, v.y, s_tag[q]);
      }
    }
  }
  int code = 0;
  for (int j = 0; j < P.nsubblk && !code; ++j) {
    uint2 *dst = reinterpret_cast<uint2 *>(P.out[c.r]) + (int64_t)j * P.out_sub_stride;
    const uint2 *mine = own + (int64_t)gi * P.istride + (int64_t)j * P.sub_stride;
    for (int64_t e = lo + threadIdx.x; e < hi && !code; e += nt) {
      uint4 w[MAXP];
      int qs[MAXP];
#pragma unroll
      for (int i = 0; i < MAXP; ++i) {
        int q;
        if (ORDER == O_RING) q = (gi + 1 + i) % gs;
        else if (ORDER == O_REC) q = gi ^ i;
        else q = i;
        qs[i] = q;
        if (i < gs && q != gi)
          w[i] = ll_ld(reinterpret_cast<const uint4 *>(ll_region(P, c.r, s_tag[q], c.world(q)) + PCCL_LL_HDR_BYTES) +
                       (int64_t)j * P.blk + e);
      }
      uint2 raw[MAXP];
#pragma unroll
      for (int i = 0; i < MAXP; ++i) {
        const int q = qs[i];
        raw[i] = make_uint2(0u, 0u);
        if (i >= gs) continue;
        if (q == gi) {
          raw[i] = __ldg(mine + e);
        } else {
          if (!ll_ok(w[i], s_tag[q]) && !code) {
            const char *reg = ll_region(P, c.r, s_tag[q], c.world(q));
            code = ll_wait(c, reinterpret_cast<const uint4 *>(reg + PCCL_LL_HDR_BYTES) + (int64_t)j * P.blk + e, s_tag[q],
                           w[i], reinterpret_cast<const uint4 *>(reg));
          }
          raw[i] = make_uint2(w[i].x, w[i].z);
        }
      }
      if (code) break;
      Acc acc;
      if (ORDER == O_REC) {
        Acc v[MAXP];
#pragma unroll
        for (int i = 0; i < MAXP; ++i) v[i] = R::load(raw[i]);
#pragma unroll
        for (int h = MAXP / 2; h >= 1; h >>= 1) {
          if (h < gs) {
#pragma unroll
            for (int m = 0; m < h; ++m) {
              acc_add<Acc, R::N>(v[m], v[m ^ h]);
              if (DT != DT_F32 && P.wire) v[m] = R::load(R::store(v[m]));
            }
          }
        }
        acc = v[0];
      } else if (ORDER == O_RANK) {
#pragma unroll
        for (int k = 0; k < R::N; ++k) acc.v[k] = 0.0f;
#pragma unroll
        for (int i = 0; i < MAXP; ++i)
          if (i < gs) acc_add<Acc, R::N>(acc, R::load(raw[i]));
      } else {
        acc = R::load(raw[0]);
#pragma unroll
        for (int i = 1; i < MAXP; ++i)
          if (i < gs) {
            acc_add<Acc, R::N>(acc, R::load(raw[i]));
            if (DT != DT_F32 && P.wire) acc = R::load(R::store(acc));
          }
      }
      dst[e] = R::store(acc);
    }
  }
  ll_finish(c, s_tag, code);
}

// Fold of the p values of one 8-byte unit in the named order (fold position
// i holds member q: ring q = gi + 1 + i, butterfly q = gi ^ i, rank q = i),
// rounding every partial to the storage type when `wire` — the same
// arithmetic as k_rs_direct_ll, so LL128 and LL results are bit-identical.
template <int DT, int ORDER, int MAXP>
__device__ __forceinline__ uint64_t ll_fold(const uint64_t (&u)[MAXP], int gs, int wire) {
  using R = LLU<DT>;
  using Acc = typename R::Acc;
  auto ld = [](uint64_t x) { return R::load(make_uint2((uint32_t)x, (uint32_t)(x >> 32))); };
  Acc acc;
  if (ORDER == O_REC) {
    Acc v[MAXP];
#pragma unroll
    for (int i = 0; i < MAXP; ++i) v[i] = ld(u[i]);
#pragma unroll
    for (int h = MAXP / 2; h >= 1; h >>= 1) {
      if (h < gs) {
#pragma unroll
        for (int m = 0; m < h; ++m) {
          acc_add<Acc, R::N>(v[m], v[m ^ h]);
          if (DT != DT_F32 && wire) v[m] = R::load(R::store(v[m]));
        }
      }
    }
    acc = v[0];
  } else if (ORDER == O_RANK) {
#pragma unroll
    for (int k = 0; k < R::N; ++k) acc.v[k] = 0.0f;
#pragma unroll
    for (int i = 0; i < MAXP; ++i)
      if (i < gs) acc_add<Acc, R::N>(acc, ld(u[i]));
  } else {
    acc = ld(u[0]);
#pragma unroll
    for (int i = 1; i < MAXP; ++i)
      if (i < gs) {
        acc_add<Acc, R::N>(acc, ld(u[i]));
        if (DT != DT_F32 && wire) acc = R::load(R::store(acc));
      }
  }
  const uint2 o = R::store(acc);
  return (uint64_t)o.x | ((uint64_t)o.y << 32);
}

// LL128 reduce-scatter: chunk q of my input goes to member q as LL128 lines;
// my output is folded from my own chunk and the p - 1 received line streams
// (a warp waits until all four lines of a group carry the tag, per source).
template <int DT, int ORDER, int MAXP>
__global__ void __launch_bounds__(kThreads) k_rs_direct_ll128(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  c.ll_ctr = PCCL_WCTRL_LL128;
  CtaEpilogue fin(c);
  __shared__ uint32_t s_tag[PCCL_MAXR];
  ll_tags(c, s_tag);
  ll_post_headers(c, s_tag);
  const int gs = c.gs, gi = c.gi;
  const int lane = threadIdx.x & 31, j = lane & 7;
  const int64_t words = P.blk;  // 8-byte units of one chunk
  const int64_t lines = (words + 14) / 15;
  const int64_t nw = (int64_t)P.ctas * (blockDim.x >> 5);
  const int64_t w0 = (int64_t)c.b * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t *own = reinterpret_cast<const uint64_t *>(P.send[c.r]) + P.base[c.y];
  for (int64_t g = w0; g * 4 < lines; g += nw) {
    const int64_t line = g * 4 + (lane >> 3);
    if (line >= lines) continue;
    const int64_t wa = line * 15 + 2 * j;
#pragma unroll
    for (int i = 1; i < MAXP; ++i) {
      if (i >= gs) break;
      const int q = (gi + i) % gs;
      const uint64_t *src = own + (int64_t)q * P.istride;
      const uint64_t a = wa < words ? src[wa] : 0ull;
      const uint64_t b = (j < 7 && wa + 1 < words) ? src[wa + 1] : (uint64_t)s_tag[q];
      uint64_t *d = reinterpret_cast<uint64_t *>(ll128_region(P, c.world(q), s_tag[q], c.r) + PCCL_LL_HDR_BYTES);
      st_line16(d + line * 16 + 2 * j, a, j < 7 ? b : (uint64_t)s_tag[q]);
    }
  }
  uint64_t *dst = reinterpret_cast<uint64_t *>(P.out[c.r]);
  const uint64_t *mine = own + (int64_t)gi * P.istride;
  int code = 0;
  for (int64_t g = w0; g * 4 < lines; g += nw) {
    const int64_t line = g * 4 + (lane >> 3);
    const bool valid = line < lines;
    const int64_t wa = line * 15 + 2 * j;
    uint64_t va[MAXP], vb[MAXP];
#pragma unroll
    for (int i = 0; i < MAXP; ++i) {
      va[i] = vb[i] = 0ull;
      if (i >= gs || code) continue;
      int q;
      if (ORDER == O_RING) q = (gi + 1 + i) % gs;
      else if (ORDER == O_REC) q = gi ^ i;
      else q = i;
      if (q == gi) {
        if (valid && wa < words) va[i] = mine[wa];
        if (valid && j < 7 && wa + 1 < words) vb[i] = mine[wa + 1];
        continue;
      }
      const char *reg = ll128_region(P, c.r, s_tag[q], c.world(q));
      const uint64_t *pl = reinterpret_cast<const uint64_t *>(reg + PCCL_LL_HDR_BYTES) + (valid ? line : 0) * 16 + 2 * j;
      const uint64_t tag = s_tag[q];
      uint64_t a, b;
      uint32_t it = 0;
      while (true) {
        ld_line16(pl, a, b);
        if (__all_sync(0xffffffffu, !valid || j != 7 || b == tag)) break;
        if ((++it & 1023u) == 0) {
          int e = lane == 0 ? ll128_slow_check(c, reg, (uint32_t)tag) : 0;
          e = __shfl_sync(0xffffffffu, e, 0);
          if (e) {
            code = e;
            break;
          }
        }
      }
      va[i] = a;
      vb[i] = j < 7 ? b : 0ull;
    }
    if (code) break;
    if (valid) {
      if (wa < words) dst[wa] = ll_fold<DT, ORDER, MAXP>(va, gs, P.wire);
      if (j < 7 && wa + 1 < words) dst[wa + 1] = ll_fold<DT, ORDER, MAXP>(vb, gs, P.wire);
    }
  }
  ll_finish(c, s_tag, code);
}

// ============================================================================
// NVLS (NVLink SHARP) collectives through a multicast segment (variant 6).
// P.recv (AG) / P.send (RS) hold this rank's *multicast* mapping of the
// segment: a multimem.st there lands in every member's copy, a
// multimem.ld_reduce returns the sum of every member's copy, both executed
// by the NVSwitch. Accesses through the multicast and the unicast mapping of
// the same memory are different proxies, hence fence.proxy.alias around the
// flag handshakes.
// ============================================================================
__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }
__device__ __forceinline__ void mc_st(uint4 *p, const uint4 &v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
template <int DT> __device__ __forceinline__ uint4 mc_ld_reduce(const uint4 *p);
template <> __device__ __forceinline__ uint4 mc_ld_reduce<DT_BF16>(const uint4 *p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
template <> __device__ __forceinline__ uint4 mc_ld_reduce<DT_F16>(const uint4 *p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
template <> __device__ __forceinline__ uint4 mc_ld_reduce<DT_F32>(const uint4 *p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// All-gather: entry = "my output may be overwritten", then every rank
// multicasts its block once, then "my block has landed everywhere".
__global__ void __launch_bounds__(kThreads) k_nvls_ag(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const uint32_t peers = ((1u << c.gs) - 1) & ~(1u << c.gi);
  cta_signal_entry(c, peers);
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  if (!cta_wait_mask(c, peers, 0)) return;
  fence_proxy_alias();
  const uint4 *src = reinterpret_cast<const uint4 *>(P.send[c.r]);
  uint4 *mc = reinterpret_cast<uint4 *>(P.recv[c.r]) + P.base[c.y] + (int64_t)c.gi * P.istride;
  const int nt = blockDim.x;
  for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)kUnroll * nt) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + (int64_t)u * nt < hi) v[u] = __ldg(src + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + (int64_t)u * nt < hi) mc_st(mc + i + (int64_t)u * nt, v[u]);
  }
  // every thread orders its multicast stores (proxy fence); the CTA barrier
  // plus the system-scope release of the "landed" flags publishes them
  fence_proxy_alias();
  cta_signal_mask(c, peers, 1);
  if (!cta_wait_mask(c, peers, 1)) return;
  fence_proxy_alias();
}

// Reduce-scatter: entry = "my input is in my copy of the segment", then
// chunk gi is read through the switch as the sum over all members (fp32
// accumulation for bf16 / fp16), exit = "I have finished reading yours".
template <int DT>
__global__ void __launch_bounds__(kThreads) k_nvls_rs(const __grid_constant__ LaunchParams P) {
  Ctx c = make_ctx(P);
  CtaEpilogue fin(c);
  const uint32_t peers = ((1u << c.gs) - 1) & ~(1u << c.gi);
  cta_signal_entry(c, peers);
  int64_t lo, hi;
  split32(P.blk, P.ctas, c.b, lo, hi);
  if (!cta_wait_mask(c, peers, 0)) return;
  fence_proxy_alias();
  const uint4 *mc = reinterpret_cast<const uint4 *>(P.send[c.r]) + P.base[c.y] + (int64_t)c.gi * P.istride;
  uint4 *dst = reinterpret_cast<uint4 *>(P.out[c.r]);
  const int nt = blockDim.x;
  for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)kUnroll * nt) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + (int64_t)u * nt < hi) v[u] = mc_ld_reduce<DT>(mc + i + (int64_t)u * nt);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + (int64_t)u * nt < hi) dst[i + (int64_t)u * nt] = v[u];
  }
  fence_proxy_alias();
  cta_exit(c, peers, peers);
}

// TMA variant of the probe (modes 4 push / 5 pull): one thread per CTA moves
// its range through a shared-memory ring with cp.async.bulk (bulk loads from
// the source, bulk stores to the destination), the data path of the TMA
// collective variants.
__global__ void __launch_bounds__(kThreads) k_probe_tma(char *local, const LaunchParams P, uint32_t dst_mask,
                                                        int64_t units, int mode) {
  extern __shared__ __align__(128) char dsm[];
  int peers[PCCL_MAXR], np = 0;
  for (int q = 0; q < PCCL_MAXR; ++q)
    if ((dst_mask >> q) & 1u) peers[np++] = q;
  if (np == 0) return;
  const int q = peers[blockIdx.x % np];
  const int per_peer_ctas = (gridDim.x + np - 1 - (blockIdx.x % np)) / np;
  int64_t lo, hi;
  split32(units, per_peer_ctas, blockIdx.x / np, lo, hi);
  TmaRing R = tma_ring_setup(dsm, P.tma_stages, P.tma_tile);
  if (threadIdx.x == 0) {
    char *rem = P.recv[q] + lo * 16, *loc = local + lo * 16;
    tma_copy_segments(R, 1, [&](int, char *&d, const char *&s, int64_t &len) {
      len = (hi - lo) * 16;
      d = mode == 4 ? rem : loc;
      s = mode == 4 ? loc : rem;
    });
  }
  __syncthreads();
}

// ============================================================================
// raw NVLink probe (debug): every CTA streams 16-byte vectors to (push) or
// from (pull) the peers in dst_mask, round-robin by CTA; no flags, no order.
// ============================================================================
__global__ void __launch_bounds__(kThreads) k_probe(char *local, const LaunchParams P, uint32_t dst_mask, int64_t units,
                                                    int mode) {
  int peers[PCCL_MAXR], np = 0;
  for (int q = 0; q < PCCL_MAXR; ++q)
    if ((dst_mask >> q) & 1u) peers[np++] = q;
  if (np == 0) return;
  const int q = peers[blockIdx.x % np];
  const int per_peer_ctas = (gridDim.x + np - 1 - (blockIdx.x % np)) / np;
  const int idx = blockIdx.x / np;
  int64_t lo, hi;
  split32(units, per_peer_ctas, idx, lo, hi);
  uint4 *rem = reinterpret_cast<uint4 *>(P.recv[q]);
  uint4 *loc = reinterpret_cast<uint4 *>(local);
  const int nt = blockDim.x;
  if (mode >= 2) {  // 256-bit accesses (LDG/STG .256 on sm_100)
    V256 *rem8 = reinterpret_cast<V256 *>(P.recv[q]);
    V256 *loc8 = reinterpret_cast<V256 *>(local);
    lo >>= 1; hi >>= 1;
    for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)kUnroll * nt) {
      V256 v[kUnroll];
      if (mode == 2) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) v[u] = ld256_nc(loc8 + i + u * nt);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) st256(rem8 + i + u * nt, v[u]);
      } else {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) v[u] = ld256_cg(rem8 + i + u * nt);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) st256(loc8 + i + u * nt, v[u]);
      }
    }
  } else if (mode == 0 || mode == 6 || mode == 7) {  // 6 / 7: remote reductions (red.add f32x4 / bf16x8, sys scope)
    for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)kUnroll * nt) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) v[u] = __ldg(loc + i + u * nt);
      if (mode == 0) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) rem[i + u * nt] = v[u];
      } else if (mode == 6) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (i + u * nt < hi)
            asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(rem + i + u * nt),
                         "f"(__uint_as_float(v[u].x)), "f"(__uint_as_float(v[u].y)), "f"(__uint_as_float(v[u].z)),
                         "f"(__uint_as_float(v[u].w))
                         : "memory");
      } else {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
          if (i + u * nt < hi)
            asm volatile("red.relaxed.sys.global.add.noftz.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(rem + i + u * nt),
                         "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                         : "memory");
      }
    }
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += (int64_t)kUnroll * nt) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) v[u] = __ldcg(rem + i + u * nt);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) if (i + u * nt < hi) loc[i + u * nt] = v[u];
    }
  }
}

// ============================================================================
// device-local helpers
// ============================================================================
// Block transpose (hierarchy.py:103-126): out block (a*B + b) = in block (b*A + a)
// where the input is a B x A grid of blocks. Grid-stride over output units.
template <int U>
__global__ void __launch_bounds__(kThreads) k_shuffle(const char *in, char *out, int A, int B, int64_t blk) {
  using T = typename VecT<U>::T;
  const T *s = reinterpret_cast<const T *>(in);
  T *d = reinterpret_cast<T *>(out);
  const int64_t total = (int64_t)A * B * blk;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ob = o / blk, e = o - ob * blk;
    const int64_t a = ob / B, b = ob - a * B;
    d[o] = __ldg(s + (b * A + a) * blk + e);
  }
}

template <int DT, bool VEC>
__global__ void __launch_bounds__(kThreads) k_reduce_inplace(char *acc, const char *other, int64_t n) {
  using R = RUnit<DT, VEC>;
  using T = typename R::T;
  T *a = reinterpret_cast<T *>(acc);
  const T *b = reinterpret_cast<const T *>(other);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    typename R::Acc s = R::load(a[i]);
    acc_add<typename R::Acc, R::N>(s, R::load(__ldg(b + i)));
    a[i] = R::store(s);
  }
}

// ============================================================================
// Copy-engine all-gather handshake (ag_variant 5). One thread spins on a META
// word of my arena until it reaches `target`, bounded by the world timeout;
// on timeout or abort it records the error and floods ABORT into every
// member's META words of the group's slot, so no peer's wait is left spinning
// (a stream memory-op wait has no deadline, which is why this is a kernel).
// ============================================================================
struct CeWait {
  const uint64_t *word;
  uint64_t target;
  volatile int *err;
  volatile uint64_t *mirror;  // this rank's device-side error mirror (WCTRL [PCCL_WCTRL_ERR])
  int64_t timeout_ns;
  int gs;
  uint64_t *meta[PCCL_MAXR];  // per member: META rows of the slot in its arena
};

__global__ void k_ce_wait(const __grid_constant__ CeWait W) {
  __shared__ int s_code;
  if (threadIdx.x == 0) {
    const uint64_t t0 = global_timer_ns();
    int code = 0;
    uint32_t it = 0;
    while (true) {
      const uint64_t v = ld_acquire_sys(W.word);
      if (v & PCCL_ABORT_BIT) { code = (int)(v & 0xff); break; }
      if (v >= W.target) break;
      if ((++it & 255u) == 0) {
        if (const uint64_t e = *W.mirror) { code = (int)e; break; }
        if (global_timer_ns() - t0 > (uint64_t)W.timeout_ns) { code = 5; break; }  // PCCL_ERR_TIMEOUT
      }
    }
    if (code && *W.mirror == 0) {
      *W.mirror = (uint64_t)code;
      *W.err = code;
      __threadfence_system();
    }
    s_code = code;
  }
  __syncthreads();
  if (s_code) {
    const uint64_t v = PCCL_ABORT_BIT | (uint64_t)s_code;
    for (int m = 0; m < W.gs; ++m)
      for (int i = threadIdx.x; i < PCCL_MAXR * PCCL_MAX_CTAS; i += blockDim.x) st_relaxed_sys(W.meta[m] + i, v);
    __threadfence_system();
  }
}

}  // namespace pccl
