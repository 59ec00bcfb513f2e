/*
 * pccl_b200.h — C ABI of the B200-native all-gather / reduce-scatter path.
 *
 * Drop-in boundary for the reference's hot path (collkit):
 * the reference's Python entry points take a Communicator and a buffer and
 * move data through a tagged point-to-point transport
 * (/root/reference/pkg/src/collkit/transport/base.py:105-174). Here the
 * transport is replaced by symmetric device memory mapped over NVLink 5 /
 * NVSwitch (CUDA IPC) and the collectives are sm_100a kernels that pull peer
 * data and fuse the reduction into the load loop. Plain C types only: device
 * pointers are void*, streams are cudaStream_t passed as void*.
 *
 * Every function returns a pccl_status_t; the Python layer maps each code 1:1
 * to the reference's exception classes (collkit/errors.py:4-62).
 *
 * Threading: a world / communicator is used by one host thread at a time
 * (collkit/transport/base.py:106-111). Calls are stream-ordered and SPMD: every
 * member issues the same collectives in the same order
 * (collkit/transport/base.py:131-134), which is what keeps the per-group epoch
 * counters (the replacement for next_base_tag) in agreement without any
 * host-side coordination. Epochs live in device memory, so every collective
 * is CUDA-graph capturable (segments must be sized before capture). All
 * collectives on one WORLD must be ordered on the device (one stream, or
 * streams ordered with events), including calls on different sub-groups: the
 * staging segment and the per-rank-pair LL channels are world resources, and
 * two concurrent collectives on the same group share its epoch word, exactly
 * like two unordered NCCL calls on one communicator. Independent streams of
 * collectives need independent worlds.
 */
#ifndef PCCL_B200_H
#define PCCL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCCL_MAX_RANKS 16        /* real mode: <= 8 GPUs of one NVSwitch box; emulation: <= 16 */
#define PCCL_IPC_HANDLE_BYTES 64 /* sizeof(cudaIpcMemHandle_t) */
#define PCCL_REG_HANDLE_BYTES 80 /* allocation IPC handle + offset + allocation size */

typedef enum {
  PCCL_SUCCESS = 0,
  PCCL_ERR_INVALID_ARGUMENT = 1,   /* ValueError            (hierarchy.py:77-80)   */
  PCCL_ERR_NON_POWER_OF_TWO = 2,   /* errors.NonPowerOfTwo  (collectives.py:113)   */
  PCCL_ERR_NOT_DIVISIBLE = 3,      /* errors.NotDivisible   (collectives.py:85)    */
  PCCL_ERR_LENGTH_MISMATCH = 4,    /* errors.LengthMismatch (collectives.py:38-41) */
  PCCL_ERR_TIMEOUT = 5,            /* errors.Timeout        (sockets.py:203-212)   */
  PCCL_ERR_PEER_UNREACHABLE = 6,   /* errors.PeerUnreachable                        */
  PCCL_ERR_UNSUPPORTED = 7,        /* errors.Unsupported                            */
  PCCL_ERR_INVALID_TOPOLOGY = 8,   /* errors.InvalidTopology (topology.py:16-33)   */
  PCCL_ERR_INDEX_OUT_OF_RANGE = 9, /* errors.IndexOutOfRange                        */
  PCCL_ERR_CUDA = 10,              /* errors.CollkitError: CUDA runtime failure     */
  PCCL_ERR_OUT_OF_MEMORY = 11,     /* staging segment too small: grow and retry     */
} pccl_status_t;

typedef enum {
  PCCL_FLOAT32 = 0,
  PCCL_BFLOAT16 = 1,
  PCCL_FLOAT16 = 2,
  PCCL_UINT8 = 3, /* all-gather only */
  PCCL_INT32 = 4, /* all-gather only */
  PCCL_INT64 = 5, /* all-gather only */
  PCCL_FLOAT64 = 6 /* all-gather only */
} pccl_dtype_t;

typedef enum {
  PCCL_ALGO_DIRECT = 0,    /* one step over every peer (new name) */
  PCCL_ALGO_RING = 1,      /* ring_all_gather / ring_reduce_scatter                 */
  PCCL_ALGO_RECURSIVE = 2  /* recdbl_all_gather / rechalf_reduce_scatter            */
} pccl_algo_t;

/* Reduction order of the DIRECT reduce-scatter (fp32 results are then
 * bit-identical to the named step-wise algorithm). */
typedef enum {
  PCCL_ORDER_RING = 0,      /* ((x_{c+1} + x_{c+2}) + ...) + x_c   (collectives.py:98-103)  */
  PCCL_ORDER_RECURSIVE = 1, /* recursive-halving butterfly          (collectives.py:150-164) */
  PCCL_ORDER_RANK = 2,      /* rank order from zeros                 (bench/oracles.py:12-19) */
  PCCL_ORDER_WIRE = 16      /* flag, direct only: round the partial to the storage type after every
                               add, where ring / recursive halving store theirs (bit-identical to
                               them in bf16 / fp16; fp32 is unaffected) */
} pccl_order_t;

typedef enum { PCCL_ALL_GATHER = 0, PCCL_REDUCE_SCATTER = 1 } pccl_collective_t;

typedef struct pccl_world *pccl_world_t; /* symmetric memory + flags of one box */
typedef struct pccl_comm *pccl_comm_t;   /* an ordered group of world ranks     */

/* ---- misc ------------------------------------------------------------- */
const char *pccl_error_string(int status);
int pccl_version(void);

/* ---- worlds ------------------------------------------------------------
 * Real mode: one process per GPU. pccl_world_create allocates segment 0 (the
 * flag arena); every segment must then be exported, exchanged by the caller's
 * bootstrap (torch.distributed) and imported on every rank.
 * Emulation mode: nranks ranks of one process on one device; each collective
 * runs all ranks in ONE cooperative launch (ranks = CTA rows), the same device
 * code as real mode with every "peer" pointer local.
 * Replaces: InProcessTransport / run_ranks (transport/inprocess.py:14-113). */
int pccl_world_create(int nranks, int rank, int device, pccl_world_t *out);
int pccl_emu_world_create(int nranks, int device, pccl_world_t *out);
int pccl_world_destroy(pccl_world_t w);
int pccl_world_check(pccl_world_t w);           /* device-reported error (sticky until reset) */
int pccl_world_error_detail(pccl_world_t w, int *out16); /* [8]=set,[9]=epoch,[10]=my hash,[11]=seen hash,[12]=rank,[13]=unit,[14]=seen unit,[15]=cta */
int pccl_world_reset_flags(pccl_world_t w);      /* zero flags + epochs (emulation, after an error) */
int pccl_world_set_tuning(pccl_world_t w, int ctas, int nsub, int threads);
int pccl_world_set_timeout_ms(pccl_world_t w, int64_t ms);
/* Tuning knobs by name: "ctas" (CTAs per rank, 0 = auto), "threads" (per
 * CTA, 64..512), "nsub" (pipeline sub-slices), "ag_variant" / "rs_variant" (data movement: -1 auto, 0 pull = LDG
 * from peers, 1 push = STG into peers, 2 TMA pull, 3 TMA push, 4 LL, 5 copy engine (AG ring /
 * recursive doubling, see pccl_ce_available) / pipelined push with pusher and folder CTAs (RS
 * direct), 7 work items (RS recursive), 8 LL128 (direct)), "tma_stages",
 * "tma_tile", "timeout_ms", "trace", "local_fence", "pdl", "ll_max" (direct
 * collectives use the LL protocol — flags inside 16-byte data words, no
 * handshakes — up to this many payload bytes per peer; -1 auto = 768 KiB /
 * (group size - 1), 0 off), "ll128_max" (direct collectives the LL rule does
 * not take use the LL128 line protocol — 120 payload bytes + a tag per
 * 128-byte line written by one warp instruction — up to this many payload
 * bytes per peer, capped at one region (1.875 MiB) and at 6 MiB (all-gather) /
 * 3 MiB (reduce-scatter) / (group size - 1); default: the cap, 0 off),
 * "item_kib" (direct collectives: CTAs claim work
 * items of this many KiB from a device counter instead of static slices;
 * default 0 = static; measured: no gain, see DESIGN), "staged_bytes" (statistic:
 * bytes of caller buffers that went through staging because they were not in a
 * registered segment; set 0 to reset). Unknown keys -> PCCL_ERR_INVALID_ARGUMENT. */
int pccl_world_set_param(pccl_world_t w, const char *key, int64_t value);
int pccl_world_get_param(pccl_world_t w, const char *key, int64_t *value);
/* With param "trace" = 1, every launch records per-CTA events (globaltimer ns
 * << 16 | kind << 12 | unit; kind 1 start, 2 wait done, 3 signal, 4 end, 5 exit,
 * 6 resident (before the PDL wait), 7 after the exit counter, 8 PDL release),
 * 128 words per CTA, laid out [row][cta][event]; copies the last launch's. */
int pccl_world_trace(pccl_world_t w, uint64_t *host, size_t cap_words, int *rows, int *ctas);
/* Param "trace" = K (2..8): the last K launches are kept; back = 0 is the
 * latest. Events: (t_ns << 16 | kind << 12 | unit), kinds 1 start, 2 wait
 * done, 3 signal, 4 exit-barrier done, 5 CTA exit. Diagnostics only. */
int pccl_world_trace_at(pccl_world_t w, int back, uint64_t *host, size_t cap_words, int *rows, int *ctas);

/* ---- symmetric segments ---------------------------------------------- */
int pccl_segment_create(pccl_world_t w, size_t bytes, int *seg_id);
int pccl_segment_export(pccl_world_t w, int seg_id, void *handle_out /* PCCL_IPC_HANDLE_BYTES */);
/* Registration of caller-owned device memory (e.g. a torch caching-allocator
 * tensor) as a segment, collectively: every rank registers its own buffer of
 * the same size, exports PCCL_REG_HANDLE_BYTES (the IPC handle of the cudaMalloc
 * allocation containing it + the offset), the bootstrap exchanges them and
 * every rank imports all (peer allocations are mapped once per process and
 * reference counted). Collectives on registered buffers are zero-copy;
 * pccl_segment_destroy unregisters (the memory stays the caller's). VMM /
 * expandable-segment memory has no IPC handle: PCCL_ERR_UNSUPPORTED. */
int pccl_segment_register(pccl_world_t w, void *ptr, size_t bytes, int *seg_id);
int pccl_segment_register_export(pccl_world_t w, int seg_id, void *handle_out /* PCCL_REG_HANDLE_BYTES */);
int pccl_segment_register_import(pccl_world_t w, int seg_id, const void *handles /* nranks x REG_HANDLE */);
int pccl_emu_segment_register(pccl_world_t w, void *const *ptrs /* nranks */, size_t bytes, int *seg_id);
int pccl_segment_import(pccl_world_t w, int seg_id, const void *handles /* nranks * 64 */);
int pccl_segment_ptr(pccl_world_t w, int seg_id, int rank, void **ptr, size_t *bytes);
int pccl_segment_destroy(pccl_world_t w, int seg_id);
int pccl_world_set_staging(pccl_world_t w, int seg_id);
/* Staging bytes a call may need (depends only on SPMD-uniform args);
 * algo 3 = hierarchical (N*M = group_size). */
size_t pccl_staging_bytes(int collective, int algo, int group_size, size_t count, int dtype);

/* ---- communicators ------------------------------------------------------
 * Replaces Communicator(...) and Communicator.subgroup (transport/base.py:113-174).
 * members are world ranks; comm_id is informational (hierarchy.py:31-38); the
 * flag slot and epoch are keyed by the member set, so re-created
 * sub-communicators keep agreeing epochs. Real mode: the caller's rank must be
 * a member (else PCCL_ERR_INDEX_OUT_OF_RANGE). */
int pccl_comm_create(pccl_world_t w, const int *members, int nmembers, int comm_id, pccl_comm_t *out);
int pccl_comm_destroy(pccl_comm_t c);
int pccl_comm_size(pccl_comm_t c, int *size);
int pccl_comm_rank(pccl_comm_t c, int *rank);
/* Completed-call counter of the group, read from member `member`'s device
 * memory (real mode: this rank only). Equal on every member between calls. */
int pccl_comm_epoch(pccl_comm_t c, int member, uint64_t *epoch);

/* ---- flat collectives (real mode: this rank's buffers) -----------------
 * pccl_all_gather replaces ring_all_gather / recdbl_all_gather
 *   (collectives.py:55-76, 107-129): recv[g*count ..] = send of group rank g.
 * pccl_reduce_scatter replaces ring_reduce_scatter / rechalf_reduce_scatter
 *   (collectives.py:79-104, 132-165): recv = chunk `rank` of the sum, chunk
 *   length recvcount; order applies to PCCL_ALGO_DIRECT only. */
int pccl_all_gather(pccl_comm_t c, int algo, const void *send, void *recv, size_t count, int dtype,
                    void *stream);
int pccl_reduce_scatter(pccl_comm_t c, int algo, int order, const void *send, void *recv, size_t recvcount,
                        int dtype, void *stream);

/* ---- point-to-point (transport/base.py:140-152) ----------------------------
 * Tagged messages between group ranks with exact (source, tag) FIFO matching.
 * pccl_send returns once the message sits in the destination's mailbox ring
 * (it never waits for a matching receive; with a full ring it drains its own
 * incoming rings while waiting, so symmetric exchanges cannot deadlock).
 * pccl_recv blocks until a message from `src` with `tag` is complete; buf ==
 * NULL probes (returns its size in *bytes and leaves it queued); a buffer
 * smaller than the message -> PCCL_ERR_LENGTH_MISMATCH (message kept). `host`
 * = 1: buf is host memory. `me` is the caller's group rank (real mode: must
 * be this process's). Host-driven control path, timeout = the world timeout. */
int pccl_send(pccl_comm_t c, int me, int dst, int64_t tag, const void *buf, size_t bytes, int host);
int pccl_recv(pccl_comm_t c, int me, int src, int64_t tag, void *buf, size_t cap, int host, size_t *bytes);

/* ---- hierarchical (hierarchy.py:158-195), world of N x M virtual nodes --- */
int pccl_hier_all_gather(pccl_world_t w, int N, int M, int inter_algo, const void *send, void *recv, size_t count,
                         int dtype, void *stream);
int pccl_hier_reduce_scatter(pccl_world_t w, int N, int M, int inter_algo, const void *send, void *recv,
                             size_t recvcount, int dtype, void *stream);
/* The same over any communicator of N x M members (hierarchy.py:129-134:
 * only the size must match the topology); topology rank g = member g. */
int pccl_hier_all_gather_comm(pccl_comm_t c, int N, int M, int inter_algo, const void *send, void *recv,
                              size_t count, int dtype, void *stream);
int pccl_hier_reduce_scatter_comm(pccl_comm_t c, int N, int M, int inter_algo, const void *send, void *recv,
                                  size_t recvcount, int dtype, void *stream);

/* ---- emulation-mode variants: per-member pointer arrays, one launch ----- */
int pccl_emu_all_gather(pccl_comm_t c, int algo, const void *const *sends, void *const *recvs, size_t count,
                        int dtype, void *stream);
int pccl_emu_reduce_scatter(pccl_comm_t c, int algo, int order, const void *const *sends, void *const *recvs,
                            size_t recvcount, int dtype, void *stream);
int pccl_emu_hier_all_gather(pccl_world_t w, int N, int M, int inter_algo, const void *const *sends,
                             void *const *recvs, size_t count, int dtype, void *stream);
int pccl_emu_hier_reduce_scatter(pccl_world_t w, int N, int M, int inter_algo, const void *const *sends,
                                 void *const *recvs, size_t recvcount, int dtype, void *stream);
int pccl_emu_hier_all_gather_comm(pccl_comm_t c, int N, int M, int inter_algo, const void *const *sends,
                                  void *const *recvs, size_t count, int dtype, void *stream);
int pccl_emu_hier_reduce_scatter_comm(pccl_comm_t c, int N, int M, int inter_algo, const void *const *sends,
                                      void *const *recvs, size_t recvcount, int dtype, void *stream);
/* Test hook: perturb one member's call signature so the device-side
 * cross-rank check must raise LengthMismatch (tests/test_collectives.py:172-175). */
int pccl_emu_debug_meta_skew(pccl_world_t w, int rank, uint32_t xor_mask);

/* Debug probe: raw NVLink throughput without any synchronisation. mode 0:
 * this rank stores `bytes` into each peer in dst_mask (second half of their
 * segment seg_id), mode 1: loads from them. */
int pccl_probe(pccl_world_t w, int seg_id, int mode, uint32_t dst_mask, size_t bytes, int ctas, void *stream);

/* ---- device-local helpers ----------------------------------------------- */
/* direction 0: shuffle_local_major_to_global, 1: shuffle_global_to_local_major
 * (hierarchy.py:103-126); out-of-place block transpose of N*M blocks. */
int pccl_shuffle(int direction, const void *in, void *out, int N, int M, size_t block_len, int dtype, void *stream);
/* reduce_inplace (collectives.py:45-52): acc[i] = acc[i] + other[i]. */
int pccl_reduce_inplace(void *acc, const void *other, size_t count, int dtype, void *stream);
/* Stream-ordered strided copy between host and device memory (any
 * direction, cudaMemcpy2DAsync semantics): `height` rows of `width` bytes,
 * row pitches in bytes. The host-buffer path of the collectives uses it to
 * move one slice of every chunk / block per call, so host<->device copies of
 * slice k+1 overlap the collective on slice k (pipelined e2e path). */
/* 1 when the copy-engine all-gather (param ag_variant = 5) can run on this
 * device: stream memory operations (64-bit) are available. The variant takes
 * ring / recursive doubling into a registered (symmetric) output outside
 * stream capture, in real mode; any other call falls back to the kernels. */
int pccl_ce_available(int device);

/* NVLS (NVLink SHARP multicast) segments and collectives. A multicast
 * segment is one switch multicast object spanning every device of the world,
 * with each rank's physical memory bound to it and mapped twice (unicast:
 * plain access to my copy; multicast: multimem ops). Setup is collective:
 * one rank pccl_nvls_create()s the object and passes the returned POSIX file
 * descriptor to the others (SCM_RIGHTS), which pccl_nvls_import() it; then
 * every rank pccl_nvls_add_device(), a barrier, every rank pccl_nvls_bind().
 * The collectives run over a world-spanning communicator; offsets, sizes
 * and pointers must be 16-byte aligned. AG: each rank multicasts its block
 * (multimem.st) into out_offset + g * count of every rank's copy. RS: each
 * rank's input sits at in_offset of its copy; chunk g is read as the switch's
 * sum over all copies (multimem.ld_reduce, fp32 accumulation for bf16 /
 * fp16) and stored to recv. The switch's summation order is not the
 * reference's, so the RS is for bf16 / fp16 training traffic, not for fp32
 * order parity. */
int pccl_nvls_supported(pccl_world_t w);
int pccl_nvls_create(pccl_world_t w, size_t bytes, size_t *alloc_bytes, int *fd, int *nvls_id);
int pccl_nvls_import(pccl_world_t w, int fd, size_t alloc_bytes, int *nvls_id);
int pccl_nvls_add_device(pccl_world_t w, int nvls_id);
int pccl_nvls_bind(pccl_world_t w, int nvls_id);
int pccl_nvls_ptr(pccl_world_t w, int nvls_id, void **unicast, void **multicast, size_t *bytes);
int pccl_nvls_destroy(pccl_world_t w, int nvls_id);
int pccl_nvls_all_gather(pccl_comm_t c, int nvls_id, const void *send, size_t out_offset, size_t count, int dtype,
                         void *stream);
int pccl_nvls_reduce_scatter(pccl_comm_t c, int nvls_id, size_t in_offset, void *recv, size_t recvcount, int dtype,
                             void *stream);
int pccl_copy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t height, void *stream);

/* ---- schedule introspection (host only, no GPU needed) -------------------
 * The step structure the kernels execute, as (step, src_world, dst_world,
 * nbytes) rows: the data that dst pulls from src in that step. Mirrors
 * simnet.build_schedule (simnet.py:326-345). m_bytes = AG output / RS input
 * per rank. Returns PCCL_ERR_OUT_OF_MEMORY if cap rows are not enough. */
int pccl_schedule(int collective, int algo, int inter_algo, int N, int M, size_t m_bytes, int64_t *rows, int cap,
                  int *nrows);

#ifdef __cplusplus
}
#endif
#endif /* PCCL_B200_H */
