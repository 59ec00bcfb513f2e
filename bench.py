"""Benchmark: reduce-scatter / all-gather bus bandwidth on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1]): reduce-scatter, bf16, 128 MiB
input per rank, recursive halving with the reduction fused into the peer-load
kernel. One *step* = one collective call. Metric: bus bandwidth
busbw = (S / t) * (p - 1) / p in GB/s (1e9 B/s), t = device time per call, max
over ranks.

* ``--gpus 1``: the reference's own shape, 8 *simulated* ranks (configs[0]
  "8 simulated ranks"), emulated on one B200: all eight ranks run in one
  cooperative launch of the same kernels, peer traffic is local HBM, so the
  roofline is HBM.
* ``--gpus N`` (N > 1): p = N real ranks, one process per GPU, over CUDA-IPC
  peer memory on NVLink 5 / NVSwitch; roofline = NVLink. Launched by the
  driver under torchrun (WORLD_SIZE == N); a plain ``python bench.py --gpus N``
  re-executes itself under ``torch.distributed.run`` with N processes. A
  world larger than the visible GPU count is refused (ranks never share a
  GPU). NCCL on the same bytes is timed beside it (default and
  ``NCCL_NVLS_ENABLE=0``, the latter in a child job of its own).

Every timed collective is VERIFIED afterwards: the inputs come from seeded
per-rank generators, each rank regenerates its peers' inputs on its own device
and recomputes its output with a torch restatement of the algorithm's
reduction order (``expected_rs`` below; bf16 partials rounded per step for the
step-wise algorithms exactly as the kernels store them), and compares bit for
bit. ``"verified": true`` on the line means the headline call and every extra
matched.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port of collkit's rechalf_reduce_scatter, ``oracle/``) on the host
cores over the same element count, in fp32 (the reference has no bf16).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "all-gather & reduce-scatter bus GB/s (64–256 MB) at 2/4/8 B200 vs 900 GB/s"
NVLINK_MEASURED_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (fallback; nominal 900)
NVLINK_NOMINAL_GBS = 900.0
# raw traffic-pattern ceilings (tools/probe.py, profiles/r1_engine_probe_p4.md): every
# reduce-scatter pulls (LDG from the peers) when its input is symmetric
PATTERN_CEILING_GBS = {"recursive": 642.0, "ring": 642.0, "direct": 634.0}
# the same kernel at 1 GiB (fixed per-call costs < 2 %): its data phase's own
# asymptote, RS bf16 (profiles/r2_sweep_p{2,4}.csv)
ASYMPTOTE_1GIB_GBS = {(2, "direct"): 657.4, (2, "ring"): 657.7, (2, "recursive"): 658.4,
                      (4, "direct"): 658.6, (4, "ring"): 661.1, (4, "recursive"): 659.5}
EMU_RANKS = 8
SEED = 20250425
P7 = 12 * 4096 * 4096 + 13 * 4096  # GPT-3-style 7B per-layer params (12h^2 + 13h, h = 4096)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def config_for(args, p: int, real: bool) -> dict:
    """The workload description; identical on the reference arm's line."""
    return {
        "workload": (f"reduce-scatter {args.dtype}, {args.size_mib} MiB input/rank, {args.algo}, p={p} "
                     + ("GPUs over NVLink/NVSwitch" if real else "simulated ranks (emulated on 1 B200 when GPU)")),
        "collective": "reduce_scatter",
        "algorithm": args.algo,
        "p": p,
        "S_bytes": args.size_mib << 20,
        "elements_per_rank": (args.size_mib << 20) // (2 if args.dtype == "bf16" else 4),
        "parallelism": f"dp{p}" if real else "emulated-8-ranks-1gpu",
        "l2": "inputs larger than L2 (per-rank input 128 MiB > 126 MB L2)",
    }


# ---------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------
class Clocks:
    """SM clock + throttle reasons sampled every 50 ms through NVML while the
    load runs (nvidia-smi with the reasons query only manages ~1 sample per
    few seconds). Device index = the CUDA ordinal; CUDA_VISIBLE_DEVICES is
    honoured by mapping through the PCI bus id."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._thread = None
        self._err = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            try:
                props = torch.cuda.get_device_properties(self.device)
                bus = f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:{props.pci_device_id:02X}.0"
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:  # noqa: BLE001 - fall back to the NVML index
                self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self._nv = pynvml
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception as exc:  # noqa: BLE001 - clocks are diagnostics
            self._err = repr(exc)[:200]
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((sm, rs))
            except Exception as exc:  # noqa: BLE001
                self._err = repr(exc)[:200]
                return
            time.sleep(0.05)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"], "samples": 0, "error": self._err}
        sm = [s for s, _ in self.samples]
        reasons = sorted({name for _, r in self.samples for name, attr in self.REASONS.items()
                          if r & getattr(self._nv, attr)})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self._max, "reasons": reasons,
                "samples": len(self.samples), "source": "NVML, 50 ms, during the soak + warm-up + timed steps"}


# ---------------------------------------------------------------------------
# CPU reference arm / baseline (oracle port of collkit, test infrastructure)
# ---------------------------------------------------------------------------
def cpu_reference(p: int, elems: int, algo: str, steps: int, warmup: int):
    """Time the reference algorithm's CPU restatement on this host's cores:
    p simulated ranks of ``elems`` fp32 elements each (the reference computes
    in fp32 only, collectives.py:26-29), the per-step work of every rank split
    over host threads by element range (numpy releases the GIL in its
    kernels; elementwise folds keep every element's reduction order)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import collectives as oc

    n = elems // p
    rng = np.random.default_rng(0)
    # the reference's sweep inputs: integer-valued fp32 in [-1024, 1024] (sweep.py:133-136)
    ins = [rng.integers(-1024, 1025, size=n * p).astype(np.float32) for _ in range(p)]
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        threads = os.cpu_count() or 1
    threads = max(1, min(threads, n // 16384 or 1))
    pool = ThreadPoolExecutor(max_workers=threads)
    fn = oc.rechalf_reduce_scatter if algo == "recursive" else oc.ring_reduce_scatter
    bounds = np.linspace(0, n, threads + 1).astype(int)

    def run(i):
        lo, hi = bounds[i], bounds[i + 1]
        sub = [np.concatenate([x[c * n + lo : c * n + hi] for c in range(p)]) for x in ins]
        return fn(sub, "f32")

    def one_call():
        list(pool.map(run, range(threads)))

    for _ in range(warmup):
        one_call()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        one_call()
        times.append(time.perf_counter() - t0)
    pool.shutdown()
    return statistics.mean(times), threads


# ---------------------------------------------------------------------------
# verification: torch restatement of the reduction orders (checker only)
# ---------------------------------------------------------------------------
def _ring_order(p: int, c: int) -> list:
    return [(c + 1 + i) % p for i in range(p)]


def expected_rs(leaves: list, c: int, algo: str, order: str = "ring", grid=None, inter: str = "ring"):
    """Chunk c of the reduce-scatter of the p leaves (leaves[q] = rank q's
    chunk c), in the order the named algorithm adds them:

    * ``ring``: left fold x_{c+1} + ... + x_c, partial stored (rounded to the
      storage dtype) after every add (collectives.py:79-104);
    * ``recursive``: butterfly T_{k+1}(i) = T_k(i) + T_k(i ^ p >> (k+1)),
      rounded per step (collectives.py:132-165);
    * ``direct``: fp32 accumulation in ``order`` (ring / recursive / rank),
      rounded once;
    * ``hierarchical`` (grid = (N, M)): inner ring over local ranks, then
      the outer ring / butterfly over nodes, rounded per step
      (hierarchy.py:176-195).
    """
    p = len(leaves)
    dt = leaves[0].dtype
    f = [x.float() for x in leaves]
    wire = algo != "direct" and dt != torch.float32

    def add(a, b):
        s = a + b
        return s.to(dt).float() if wire else s

    def ring_fold(vals, cc):
        o = _ring_order(len(vals), cc)
        acc = vals[o[0]]
        for i in o[1:]:
            acc = add(acc, vals[i])
        return acc

    def butterfly(vals, cc):
        t = list(vals)
        h = len(t) >> 1
        while h >= 1:
            t = [add(t[i], t[i ^ h]) for i in range(len(t))]
            h >>= 1
        return t[cc]

    if algo == "hierarchical":
        N, M = grid
        node, j = divmod(c, M)
        parts = [ring_fold([f[nd * M + l] for l in range(M)], j) for nd in range(N)]
        acc = butterfly(parts, node) if inter == "recursive" else ring_fold(parts, node)
    elif algo == "ring" or (algo == "direct" and order == "ring"):
        acc = ring_fold(f, c)
    elif algo == "recursive" or (algo == "direct" and order == "recursive"):
        acc = butterfly(f, c)
    elif order == "rank":
        acc = torch.zeros_like(f[0])
        for v in f:
            acc = add(acc, v)
    else:
        raise ValueError(f"unknown algorithm/order {algo}/{order}")
    return acc.to(dt)


def _bits_equal(a: torch.Tensor, b: torch.Tensor) -> bool:
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    iv = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[a.element_size()]
    return bool(torch.equal(a.contiguous().view(iv), b.contiguous().view(iv)))


def seeded_fill(t: torch.Tensor, seed: int) -> None:
    g = torch.Generator(device=t.device)
    g.manual_seed(seed)
    t.normal_(generator=g)


# ---------------------------------------------------------------------------
# the rig: real ranks (one process per GPU) or p ranks emulated on one GPU
# ---------------------------------------------------------------------------
class Rig:
    def __init__(self, real: bool, p: int, rank: int, dev: torch.device, dist=None, comm=None):
        import paper_2504_18658_b200 as pkg
        from paper_2504_18658_b200 import _lib
        from paper_2504_18658_b200.communicator import _emu_group, emulated_world

        self.pkg, self._lib, self.L = pkg, _lib, _lib.lib()
        self.real, self.p, self.rank, self.dev, self.dist = real, p, rank, dev, dist
        self.stream = torch.cuda.current_stream(dev)
        if real:
            self.comm = comm if comm is not None else pkg.init_from_torch(device=dev.index)
            self.world = self.comm.world
            self.ghandle = self.comm.handle
        else:
            self.comm = None
            self.world = emulated_world(p, dev.index)
            self.group, _ = _emu_group(self.world, tuple(range(p)), 0)
        self._seed = SEED

    # -- buffers ---------------------------------------------------------
    def sym(self, numel: int, dtype):
        """Symmetric buffer: this rank's tensor (real) or one per rank (emulated)."""
        return self.world.empty(numel, dtype)

    def tensors(self, buf) -> dict:
        """{world rank: tensor} of the ranks this process executes."""
        return {self.rank: buf} if self.real else dict(enumerate(buf))

    def ptr(self, buf):
        return buf.data_ptr() if self.real else self._lib.ptr_array([t.data_ptr() for t in buf])

    def new_seed(self) -> int:
        self._seed += 1000
        return self._seed

    def fill(self, buf, seed: int) -> None:
        for r, t in self.tensors(buf).items():
            seeded_fill(t, seed + r)

    def inputs(self, buf, seed: int, numel: int, dtype, q: int):
        """Rank q's input (regenerated on this device in real mode)."""
        if not self.real:
            return buf[q]
        if q == self.rank:
            return buf
        t = torch.empty(numel, dtype=dtype, device=self.dev)
        seeded_fill(t, seed + q)
        return t

    # -- calls -----------------------------------------------------------
    def staging(self, coll: int, algo: int, n: int, code: int) -> None:
        self.world.ensure_staging(int(self.L.pccl_staging_bytes(coll, algo, self.p, n, code)))

    def rs(self, algo: str, order: str, bin_, bout, n: int, code: int):
        a, o = self._lib.ALGOS[algo], self._lib.ORDERS[order]
        self.staging(1, a, n, code)
        si, so, s = self.ptr(bin_), self.ptr(bout), self.stream.cuda_stream
        if self.real:
            return lambda: self._lib.check(self.L.pccl_reduce_scatter(self.ghandle, a, o, si, so, n, code, s))
        return lambda: self._lib.check(self.L.pccl_emu_reduce_scatter(self.group.handle, a, o, si, so, n, code, s))

    def ag(self, algo: str, bin_, bout, n: int, code: int):
        a = self._lib.ALGOS[algo]
        self.staging(0, a, n, code)
        si, so, s = self.ptr(bin_), self.ptr(bout), self.stream.cuda_stream
        if self.real:
            return lambda: self._lib.check(self.L.pccl_all_gather(self.ghandle, a, si, so, n, code, s))
        return lambda: self._lib.check(self.L.pccl_emu_all_gather(self.group.handle, a, si, so, n, code, s))

    def hier(self, coll: str, N: int, M: int, inter: str, bin_, bout, n: int, code: int):
        ia = self._lib.ALGOS[inter]
        self.staging(1, 3, n, code)
        si, so, s, h = self.ptr(bin_), self.ptr(bout), self.stream.cuda_stream, self.world.handle
        L = self.L
        if coll == "ag":
            fn = L.pccl_hier_all_gather if self.real else L.pccl_emu_hier_all_gather
        else:
            fn = L.pccl_hier_reduce_scatter if self.real else L.pccl_emu_hier_reduce_scatter
        return lambda: self._lib.check(fn(h, N, M, ia, si, so, n, code, s))

    # -- cross-rank reductions ----------------------------------------------
    def barrier(self):
        torch.cuda.synchronize()
        if self.real:
            self.dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if not self.real:
            return x
        tt = torch.tensor([x], device=self.dev, dtype=torch.float64)
        self.dist.all_reduce(tt, op=self.dist.ReduceOp.MAX)
        return float(tt.item())

    def all_ok(self, ok: bool) -> bool:
        if not self.real:
            return ok
        tt = torch.tensor([1 if ok else 0], device=self.dev, dtype=torch.int32)
        self.dist.all_reduce(tt, op=self.dist.ReduceOp.MIN)
        return bool(tt.item())

    # -- verification --------------------------------------------------------
    def verify_rs(self, bin_, bout, seed: int, n: int, dtype, algo: str, order: str = "ring", grid=None,
                  inter: str = "ring") -> bool:
        ok = True
        for r, out in self.tensors(bout).items():
            leaves = []
            for q in range(self.p):
                x = self.inputs(bin_, seed, n * self.p, dtype, q)
                leaves.append(x[r * n : (r + 1) * n].clone())
                del x
            want = expected_rs(leaves, r, algo, order, grid, inter)
            ok &= _bits_equal(out[:n], want)
        torch.cuda.synchronize()
        return self.all_ok(ok)

    def verify_ag(self, bin_, bout, seed: int, n: int, dtype) -> bool:
        ok = True
        for r, out in self.tensors(bout).items():
            for q in range(self.p):
                ok &= _bits_equal(out[q * n : (q + 1) * n], self.inputs(bin_, seed, n, dtype, q)[:n])
        torch.cuda.synchronize()
        return self.all_ok(ok)

    def generator_reproducible(self, buf, seed: int, numel: int, dtype) -> bool:
        """Regenerating an input must reproduce it bit for bit (else the
        verification would compare against something else)."""
        for r, t in self.tensors(buf).items():
            x = torch.empty(numel, dtype=dtype, device=self.dev)
            seeded_fill(x, seed + r)
            if not _bits_equal(x, t[:numel]):
                return False
        return True


def busbw(s_bytes: int, p: int, seconds: float) -> float:
    return s_bytes * (p - 1) / p / seconds / 1e9


def rs_algorithmic_hbm_bytes(algo: str, p: int, chunk_bytes: int) -> int:
    """HBM bytes one emulated launch must move (all p ranks' traffic is local)."""
    if algo == "direct":
        per_rank = p * chunk_bytes + chunk_bytes          # read p chunks, write 1
    else:
        per_rank = 3 * (p - 1) * chunk_bytes              # each step: read local + peer, write
    return per_rank * p


def time_calls(call, steps: int, stream) -> float:
    """Average seconds per call over `steps` back-to-back calls on `stream`.

    One untimed call goes first: it is a device-side rendezvous of all ranks,
    so the start event is recorded when every rank's stream has reached the
    timed region. Without it the slowest rank's host leaving the barrier late
    (scheduling jitter, up to ~1 ms on these hosts) lands in the other ranks'
    first timed call."""
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    call()
    e0.record(stream)
    for _ in range(steps):
        call()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / steps


def time_graph(rig, make_call, steps: int) -> float:
    """Seconds per call with the same `steps` calls captured in ONE CUDA graph
    and replayed (the collectives are capture-safe: device-side epochs). On
    this driver an eagerly launched kernel that touched peer memory pays
    ~3.6 us at its boundary that a kernel inside a graph does not
    (tools/pdl_probe.cu, profiles/r2_launch_boundary.md)."""
    side = torch.cuda.Stream(rig.dev)
    saved = rig.stream
    rig.stream = side
    try:
        call = make_call()
    finally:
        rig.stream = saved
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(steps):
            call()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    rig.barrier()
    with torch.cuda.stream(side):
        call()  # device-side rendezvous of the ranks, as in time_calls
        e0.record(side)
        g.replay()
        e1.record(side)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / steps


def run_gpu(args):
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    real = world_size > 1
    ndev = torch.cuda.device_count()
    if local_rank >= ndev:  # ranks never time-share a GPU (spinning peers on one device can hang it)
        raise SystemExit(f"rank {rank}: local rank {local_rank} but only {ndev} visible GPU(s); "
                         "one process per GPU is required")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if real:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    p = world_size if real else EMU_RANKS
    S = args.size_mib << 20
    dtype = {"bf16": torch.bfloat16, "f32": torch.float32}[args.dtype]
    es = torch.empty(0, dtype=dtype).element_size()
    n = S // es // p
    rig = Rig(real, p, rank, dev, dist)
    _lib = rig._lib
    code = _lib.DTYPES[args.dtype]
    stream = rig.stream

    # "auto": the library's measured selector; a GPU count the shipped table
    # does not cover is calibrated on this box first (collective, untimed)
    algo = args.algo
    selection = "explicit (BASELINE configs[1]: recursive halving)" if algo == "recursive" else "explicit"
    autotuned = None
    if real:
        from paper_2504_18658_b200 import selector, tuning

        missing = [c for c in ("reduce_scatter", "all_gather") if not tuning.has_entries(c, p)]
        if args.retune or (missing and not args.profile):
            autotuned = {}
            for coll in (missing if not args.retune else ("reduce_scatter", "all_gather")):
                dt_t = torch.bfloat16 if coll == "reduce_scatter" else torch.float32
                for S_t in (64 << 20, 128 << 20, 256 << 20):
                    res = tuning.autotune(rig.comm, coll, S_t, dtype=dt_t)
                    autotuned[f"{coll}_{S_t >> 20}MiB"] = {k: round(v, 1) for k, v in res.items()}
        if algo == "auto":
            algo = selector.choose_algorithm("reduce_scatter", p, S)
            selection = "measured selector table" + (" (autotuned on this box)" if autotuned else "")
    elif algo == "auto":
        algo, selection = "recursive", "emulated N=1 headline: recursive halving"
    args.algo = algo
    order = "recursive" if algo == "recursive" else "ring"

    # ---- symmetric buffers (inputs resident in HBM, zero-copy), seeded ----
    sin, sout = rig.sym(n * p, dtype), rig.sym(n, dtype)
    seed0 = rig.new_seed()
    rig.fill(sin, seed0)
    call = rig.rs(algo, order, sin, sout, n, code)

    # ---- soak (for the clock sampler), warmup, timed region ----
    clocks = Clocks(local_rank)
    with clocks:
        # ~3 s of load for the clock sampler. The call count must be the same
        # on every rank (SPMD: each rank issues the same collectives), so it is
        # derived from a max-over-ranks estimate, never from local wall clock.
        if not args.profile:
            for _ in range(3):  # first launches load modules: keep them out of the estimate
                call()
            t_est = rig.max_over_ranks(time_calls(call, 5, stream))
            for i in range(max(20, min(60000, int(3.0 / max(t_est, 1e-6))))):
                call()
                if i % 50 == 49:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
        for _ in range(args.warmup):
            call()
        rig.barrier()
        t_call = time_calls(call, args.steps, stream)
        rig.world.check()
        rig.barrier()
    t_call = rig.max_over_ranks(t_call)
    value = busbw(S, p, t_call)
    # the output of the last timed call, checked bit for bit
    verified = rig.generator_reproducible(sin, seed0, n * p, dtype) and \
        rig.verify_rs(sin, sout, seed0, n, dtype, algo, order)
    checks = {"headline": verified}

    # the same calls captured in one CUDA graph (real mode: the launch-boundary
    # cost it removes only exists for kernels that touch peer memory)
    graph = None
    if real and not args.profile:
        try:
            t_graph = rig.max_over_ranks(time_graph(rig, lambda: rig.rs(algo, order, sin, sout, n, code),
                                                    args.steps))
            g_ok = rig.verify_rs(sin, sout, seed0, n, dtype, algo, order)
            checks["headline_graph"] = g_ok
            graph = {"value": round(busbw(S, p, t_graph), 2), "unit": "GB/s",
                     "ms_per_step": round(t_graph * 1e3, 5), "verified": g_ok, "gpu_launches": args.steps,
                     "how": "the same K calls captured in one CUDA graph and replayed (eager launches of kernels "
                            "that touch peer memory pay ~3.6 us each at the launch boundary, tools/pdl_probe.cu)"}
        except Exception as exc:  # noqa: BLE001 - a secondary number never costs the headline line
            graph = {"value": None, "error": f"{type(exc).__name__}: {exc}"[:200]}
            rig.world.check()  # a device error still surfaces

    extra = {} if args.no_extra else run_extras(args, rig, p, S, n, dtype, code, checks)

    # ---- e2e through the public API with host buffers ----
    if args.profile:
        e2e = None
    elif "error" in extra:  # a device error poisons the world: no further collectives
        e2e = {"value": None, "unit": "GB/s", "error": "skipped after: " + extra["error"][:200]}
    else:
        e2e = run_e2e(args, rig.pkg, real, p, S, dtype, dev, rig.comm, dist)

    # ---- roofline of the dominant kernel (the measured call itself) ----
    pk, src = peaks()
    if real:
        achieved = value  # algorithmic NVLink bytes per GPU per launch / launch time
        roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_MEASURED_GBS,
                "unit": "GB/s", "frac": round(achieved / NVLINK_MEASURED_GBS, 4),
                "frac_of_nominal_900": round(achieved / NVLINK_NOMINAL_GBS, 4),
                # the traffic pattern's own measured ceiling (raw 16-byte loops, no flags, p=4,
                # tools/probe.py / profiles/r1_engine_probe_p4.md)
                "pattern_ceiling": {"gbs": PATTERN_CEILING_GBS.get(algo), "frac": round(
                    achieved / PATTERN_CEILING_GBS[algo], 4) if algo in PATTERN_CEILING_GBS else None,
                    "source": "tools/probe.py raw loops at p=4: recursive / ring = bidirectional LDG pull, "
                              "direct = all-to-all LDG pull"},
                "asymptote_1gib": {"gbs": ASYMPTOTE_1GIB_GBS.get((p, algo)), "frac": round(
                    achieved / ASYMPTOTE_1GIB_GBS[(p, algo)], 4) if (p, algo) in ASYMPTOTE_1GIB_GBS else None,
                    "source": "the same kernel at 1 GiB per rank (per-call fixed costs < 2 %), "
                              "profiles/r2_sweep_p{2,4}.csv"},
                "peak_source": "B200_PROFILING.md measured peer copy (nominal 900)",
                "algorithmic_bytes_per_launch": int(S * (p - 1) / p), "traffic": None}
    else:
        hbm = rs_algorithmic_hbm_bytes(algo, p, n * es)
        achieved = hbm / t_call / 1e9
        peak = float(pk.get("hbm_gbs", 6650.0))
        traffic = args.traffic
        if traffic is None and algo == "recursive" and args.dtype == "bf16" and args.size_mib == 128:
            # dram__bytes_read.sum + dram__bytes_write.sum of this launch, ncu --set full
            # (profiles/r2_ncu_k_rs_rec_emulated.md): 1.878867 GB + 0.915568 GB
            traffic = 2794435384
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                "algorithmic_bytes_per_launch": hbm, "traffic": traffic,
                "traffic_source": "ncu --set full capture, profiles/r2_ncu_k_rs_rec_emulated.md" if traffic else None}

    cpu = None
    if rank == 0 and not real and not args.no_cpu:
        t_cpu, cores = cpu_reference(p, S // es, algo if algo != "direct" else "recursive", steps=2, warmup=1)
        cpu = {"value": round(busbw(S, p, t_cpu), 4), "unit": "GB/s", "cores": cores, "kind": "port",
               "ms_per_call": round(t_cpu * 1e3, 1),
               "sample": f"the full workload: oracle port of collkit {algo} reduce-scatter, p={p} ranks x "
                         f"{S // es} elements (the same element count, in fp32: the reference has no bf16), "
                         f"2 calls, numpy on {cores} threads; value uses the workload's S"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 2),
            "unit": "GB/s",
            "n_gpus": world_size,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(t_call * 1e3, 5),
            # busbw is a per-GPU figure by definition (the metric's "... vs 900 GB/s" per GPU);
            # the whole job moves value x ranks bus bytes per second
            "value_is": "per-GPU bus bandwidth busbw = (S/t)(p-1)/p, t = max over ranks; whole-job bus "
                        "bytes/s in aggregate_gbs",
            "aggregate_gbs": round(value * p, 1),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": args.dtype,
            "data": "synthetic (seeded standard normal per rank, resident in symmetric HBM segments)",
            "config": config_for(args, p, real),
            "selection": selection,
            "verified": all(checks.values()),
            "verification": "each rank regenerates its peers' seeded inputs on its device and recomputes its "
                            "output in the algorithm's reduction order (bench.expected_rs); bit-exact compare "
                            "of the last timed call's output, every extra likewise",
            "checks_failed": sorted(k for k, v in checks.items() if not v),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "graph_replay": graph,
            "clocks": clocks.summary(),
            "autotune": autotuned,
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if real:
        dist.barrier()
        dist.destroy_process_group()


def run_extras(args, rig, p, S, n, dtype, code, checks) -> dict:
    """The other algorithms, all-gather, the metric's 64-256 MB range,
    hierarchical (C3), FSDP 7B shapes (C5), NCCL and NVLS, every one verified."""
    extra = {}
    real, dev, stream = rig.real, rig.dev, rig.stream

    def measure(fn, k=max(5, args.steps)):
        for _ in range(3):
            fn()
        rig.barrier()
        t = time_calls(fn, k, stream)
        rig.world.check()
        return rig.max_over_ranks(t)

    def rec(tag, s_bytes, t, ok, **kw):
        extra[tag] = {"busbw_gbs": round(busbw(s_bytes, p, t), 1), "us": round(t * 1e6, 1), "verified": ok, **kw}
        checks[tag] = ok

    try:
        # every flat algorithm, both collectives, across the metric's range (64-256 MB)
        for S_r in sorted({64 << 20, S, 256 << 20}):
            for coll, dt_r, nm in (("rs", dtype, args.dtype), ("ag", torch.float32, "f32")):
                es_r = torch.empty(0, dtype=dt_r).element_size()
                n_r = S_r // es_r // p
                code_r = rig._lib.DTYPES[nm]
                c_in, c_out = (n_r * p, n_r) if coll == "rs" else (n_r, n_r * p)
                bi, bo = rig.sym(c_in, dt_r), rig.sym(c_out, dt_r)
                seed = rig.new_seed()
                rig.fill(bi, seed)
                for alg2 in ("direct", "ring", "recursive"):
                    o2 = "recursive" if alg2 == "recursive" else "ring"
                    if coll == "rs":
                        f = rig.rs(alg2, o2, bi, bo, n_r, code_r)
                        t = measure(f)
                        ok = rig.verify_rs(bi, bo, seed, n_r, dt_r, alg2, o2)
                    else:
                        f = rig.ag(alg2, bi, bo, n_r, code_r)
                        t = measure(f)
                        ok = rig.verify_ag(bi, bo, seed, n_r, dt_r)
                    rec(f"{coll}_{nm}_{S_r >> 20}MiB_{alg2}", S_r, t, ok)
                del bi, bo

        dist = rig.dist
        if real:
            nccl_ver = ".".join(map(str, torch.cuda.nccl.version()))
            for S_r, dt_r, nm in ((S, dtype, args.dtype), (64 << 20, torch.float32, "f32")):
                es_r = torch.empty(0, dtype=dt_r).element_size()
                n_r = S_r // es_r // p
                if nm == args.dtype and S_r == S:
                    nin = torch.empty(n_r * p, dtype=dt_r, device=dev).normal_()
                    nout = torch.empty(n_r, dtype=dt_r, device=dev)
                    t = measure(lambda: dist.reduce_scatter_tensor(nout, nin))
                    extra[f"nccl_rs_{nm}_{S_r >> 20}MiB"] = {"busbw_gbs": round(busbw(S_r, p, t), 1),
                                                             "us": round(t * 1e6, 1), "nccl": nccl_ver}
                    del nin, nout
                seed = rig.new_seed()
                agi = torch.empty(n_r, dtype=dt_r, device=dev)
                seeded_fill(agi, seed + rig.rank)
                ago = torch.empty(n_r * p, dtype=dt_r, device=dev)
                t = measure(lambda: dist.all_gather_into_tensor(ago, agi))
                extra[f"nccl_ag_{nm}_{S_r >> 20}MiB"] = {"busbw_gbs": round(busbw(S_r, p, t), 1),
                                                         "us": round(t * 1e6, 1), "nccl": nccl_ver,
                                                         "same_bits_as_expected": rig.verify_ag(agi, ago, seed, n_r,
                                                                                                dt_r)}
                del agi, ago

        # C3: hierarchical AG + RS, 256 MiB fp32, virtual N x M groupings
        S_h = 256 << 20
        grids = [(N, p // N) for N in (2, 4) if p % N == 0 and 1 < N < p]
        if grids:
            n_h = S_h // 4 // p
            hai, hao = rig.sym(n_h, torch.float32), rig.sym(n_h * p, torch.float32)
            hri, hro = rig.sym(n_h * p, torch.float32), rig.sym(n_h, torch.float32)
            sa, sr = rig.new_seed(), rig.new_seed()
            rig.fill(hai, sa)
            rig.fill(hri, sr)
            for (N, M) in grids:
                inter = "recursive" if N >= 4 else "ring"
                t = measure(rig.hier("ag", N, M, inter, hai, hao, n_h, 0))
                rec(f"hier_ag_f32_256MiB_{N}x{M}_{inter}", S_h, t, rig.verify_ag(hai, hao, sa, n_h, torch.float32))
                t = measure(rig.hier("rs", N, M, inter, hri, hro, n_h, 0))
                rec(f"hier_rs_f32_256MiB_{N}x{M}_{inter}", S_h, t,
                    rig.verify_rs(hri, hro, sr, n_h, torch.float32, "hierarchical", grid=(N, M), inter=inter))
            del hai, hao, hri, hro

        # C5: FSDP / ZeRO-3 GPT-3-style 7B per-layer shapes, bf16, through the
        # torch.distributed-shaped wrappers (algorithm picked by the selector)
        if real:
            pkg = rig.pkg
            n7 = P7 // p
            S7 = n7 * p * 2
            prm, full = rig.sym(n7, torch.bfloat16), rig.sym(n7 * p, torch.bfloat16)
            grad, gsh = rig.sym(n7 * p, torch.bfloat16), rig.sym(n7, torch.bfloat16)
            s_p, s_g = rig.new_seed(), rig.new_seed()
            rig.fill(prm, s_p)
            rig.fill(grad, s_g)
            rig.staging(1, 2, n7, 1)
            a_ag = pkg.choose_algorithm("all_gather", p, S7)
            a_rs = pkg.choose_algorithm("reduce_scatter", p, S7)
            t = measure(lambda: pkg.all_gather_into_tensor(full, prm, rig.comm))
            rec("fsdp7b_layer_ag_bf16", S7, t, rig.verify_ag(prm, full, s_p, n7, torch.bfloat16), bytes_out=S7,
                algorithm=a_ag)
            t = measure(lambda: pkg.reduce_scatter_tensor(gsh, grad, rig.comm))
            rec("fsdp7b_layer_rs_bf16", S7, t,
                rig.verify_rs(grad, gsh, s_g, n7, torch.bfloat16, a_rs, "ring"), bytes_in=S7, algorithm=a_rs)
            nfull = torch.empty(n7 * p, dtype=torch.bfloat16, device=dev)
            nprm = torch.empty(n7, dtype=torch.bfloat16, device=dev)
            seeded_fill(nprm, s_p + rig.rank)
            t = measure(lambda: dist.all_gather_into_tensor(nfull, nprm))
            extra["nccl_fsdp7b_layer_ag_bf16"] = {"busbw_gbs": round(busbw(S7, p, t), 1), "us": round(t * 1e6, 1),
                                                  "same_bits_as_ours": _bits_equal(nfull, full)}
            ngrad = torch.empty(n7 * p, dtype=torch.bfloat16, device=dev).normal_()
            t = measure(lambda: dist.reduce_scatter_tensor(nprm, ngrad))
            extra["nccl_fsdp7b_layer_rs_bf16"] = {"busbw_gbs": round(busbw(S7, p, t), 1), "us": round(t * 1e6, 1)}
            del nfull, nprm, ngrad, prm, full, grad, gsh

            # NVLS: switch multicast stores (AG) / switch reductions (bf16 RS)
            extra.update(run_nvls(rig, p, S, n, measure))
    except Exception as exc:  # an extra must never cost the headline line
        extra["error"] = f"{type(exc).__name__}: {exc}"[:300]
        checks["extras_completed"] = False
        if rig.rank == 0:
            print(f"[bench] extra measurements aborted: {exc!r}", file=sys.stderr, flush=True)

    if real and "error" not in extra and not args.no_nccl_child:
        extra.update(run_nccl_child(args, rig, p))
    return extra


def run_nvls(rig, p, S, n, measure) -> dict:
    from paper_2504_18658_b200 import nvls as NV

    out = {}
    try:
        if not NV.nvls_supported(rig.world):
            return {"nvls": "not supported on this box"}
        seg = NV.create_nvls_segment(rig.world, max(S, P7 * 2 + 4096))
        try:
            nx = seg.tensor(0, n * p, torch.bfloat16)
            nx.normal_()
            ny = torch.empty(n, dtype=torch.bfloat16, device=rig.dev)
            t = measure(lambda: NV.nvls_reduce_scatter(rig.comm, seg, nx, ny))
            out[f"nvls_rs_bf16_{S >> 20}MiB"] = {"busbw_gbs": round(busbw(S, p, t), 1), "us": round(t * 1e6, 1)}
            for S_a, dt_a, nm in ((64 << 20, torch.float32, "ag_f32_64MiB"),
                                  (P7 // p * p * 2, torch.bfloat16, "fsdp7b_layer_ag_bf16")):
                n_a = S_a // torch.empty(0, dtype=dt_a).element_size() // p
                seed = rig.new_seed()
                ax = torch.empty(n_a, dtype=dt_a, device=rig.dev)
                seeded_fill(ax, seed + rig.rank)
                ay = seg.tensor(0, n_a * p, dt_a)
                t = measure(lambda: NV.nvls_all_gather(rig.comm, seg, ax, ay))
                out[f"nvls_{nm}"] = {"busbw_gbs": round(busbw(S_a, p, t), 1), "us": round(t * 1e6, 1),
                                     "verified": rig.verify_ag(ax, ay, seed, n_a, dt_a)}
        finally:
            seg.close()
    except Exception as exc:  # noqa: BLE001 - optional path, never costs the rest
        out["nvls_error"] = f"{type(exc).__name__}: {exc}"[:200]
        rig.world.check()  # a device error (poisoned world) still ends the extras
    return out


def run_nccl_child(args, rig, p) -> dict:
    """NCCL with NVLS disabled: NCCL reads NCCL_NVLS_ENABLE once per process,
    so every rank runs a child job of its own (same ranks, another port)."""
    env = dict(os.environ, NCCL_NVLS_ENABLE="0", MASTER_PORT=str(int(os.environ.get("MASTER_PORT", "29500")) + 37))
    # under torchrun the env:// rendezvous would connect to the agent's store
    # instead of serving its own on the new port
    env.pop("TORCHELASTIC_USE_AGENT_STORE", None)
    cmd = [sys.executable, os.path.abspath(__file__), "--nccl-child", "--size-mib", str(args.size_mib),
           "--dtype", args.dtype, "--steps", str(max(5, args.steps))]
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=180)
        if rig.rank == 0:
            for ln in r.stdout.splitlines():
                if ln.startswith("{"):
                    return json.loads(ln)
            return {"nccl_nvls_disabled_error": (r.stderr or r.stdout)[-300:]}
    except Exception as exc:  # noqa: BLE001
        return {"nccl_nvls_disabled_error": repr(exc)[:200]}
    return {}


def nccl_child(args):
    import torch.distributed as dist

    rank, p, lr = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", lr)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    dtype = {"bf16": torch.bfloat16, "f32": torch.float32}[args.dtype]
    out = {}

    def measure(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        t = time_calls(fn, args.steps, stream)
        tt = torch.tensor([t], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    S = args.size_mib << 20
    n = S // torch.empty(0, dtype=dtype).element_size() // p
    x, y = torch.empty(n * p, dtype=dtype, device=dev).normal_(), torch.empty(n, dtype=dtype, device=dev)
    t = measure(lambda: dist.reduce_scatter_tensor(y, x))
    out[f"nccl_nvls0_rs_{args.dtype}_{args.size_mib}MiB"] = {"busbw_gbs": round(busbw(S, p, t), 1),
                                                             "us": round(t * 1e6, 1)}
    n = (64 << 20) // 4 // p
    a, b = torch.empty(n, device=dev).normal_(), torch.empty(n * p, device=dev)
    t = measure(lambda: dist.all_gather_into_tensor(b, a))
    out["nccl_nvls0_ag_f32_64MiB"] = {"busbw_gbs": round(busbw(64 << 20, p, t), 1), "us": round(t * 1e6, 1),
                                      "env": "NCCL_NVLS_ENABLE=0"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_e2e(args, pkg, real, p, S, dtype, dev, comm, dist):
    """Same metric through the public API with pinned host buffers: every step
    uploads the inputs, runs the collective and reads the result back."""
    es = torch.empty(0, dtype=dtype).element_size()
    n = S // es // p
    algo = args.algo
    fn = pkg.rechalf_reduce_scatter if algo == "recursive" else (
        pkg.ring_reduce_scatter if algo == "ring" else pkg.direct_reduce_scatter)
    steps = max(5, min(args.steps, 15))
    if real:
        x = torch.empty(n * p, dtype=dtype).normal_().pin_memory()
        for _ in range(2):
            fn(comm, x)
        torch.cuda.synchronize()
        dist.barrier()
        per = []
        for _ in range(steps):
            t0 = time.perf_counter()
            fn(comm, x)
            per.append(time.perf_counter() - t0)
        tt = torch.tensor(per, device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)  # per step: the slowest rank
        per = tt.tolist()
        h2d, d2h = n * p * es, n * es
    else:
        xs = [torch.empty(n * p, dtype=dtype).normal_().pin_memory() for _ in range(p)]
        timing = {}

        def body(c):
            for _ in range(2):
                fn(c, xs[c.rank])
            per = []
            for _ in range(steps):
                t0 = time.perf_counter()
                fn(c, xs[c.rank])
                per.append(time.perf_counter() - t0)
            if c.rank == 0:  # the emulated ranks finish each step together (one launch)
                timing["per"] = per
            return None

        pkg.run_ranks(p, body, device=dev.index)
        per = timing["per"]
        h2d, d2h = n * p * es * p, n * es * p  # all p emulated ranks' buffers cross this GPU's host link
    # host-link-bound and noisy on shared hosts (single steps up to 2x the
    # typical one): the value is the median step, the mean is reported beside it
    dt = statistics.median(per)
    mean = sum(per) / len(per)
    return {"value": round(busbw(S, p, dt), 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(dt * 1e3, 3),
            "ms_per_step_mean": round(mean * 1e3, 3), "steps": len(per), "statistic": "median step",
            "bytes_per_step_are": "per GPU" if real else "whole job (8 emulated ranks on 1 GPU)",
            "path": f"paper_2504_18658_b200.{fn.__name__}(comm, pinned host tensor) -> host tensor "
                    "(sliced, copies overlapped with the collective)"}


def run_reference(args):
    world_size = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p = world_size if world_size > 1 else EMU_RANKS
    real = world_size > 1
    if args.algo in ("auto", "direct"):  # the reference has ring and recursive halving only
        args.algo = "recursive"
    S = args.size_mib << 20
    elems = S // (2 if args.dtype == "bf16" else 4)
    t, cores = cpu_reference(p, elems, args.algo, steps=args.steps, warmup=args.warmup)
    v = busbw(S, p, t)
    sample = (f"the full workload (not a sample): oracle port of collkit {args.algo} reduce-scatter, p={p} "
              f"simulated ranks x {elems} elements per rank (the same element count as the {args.dtype} "
              f"workload; computed in fp32, the reference's only precision), numpy on {cores} host threads; "
              f"value = busbw with the workload's S = {S} bytes")
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": world_size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (integer-valued fp32, sweep.py:133-136)",
        "config": config_for(args, p, real),
        "impl": "reference",
        "elements_per_s": round(elems * p / t, 1),
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """``python bench.py --gpus N`` without a launcher: one process per GPU
    under torch.distributed.run (rank 0 prints the line)."""
    ndev = torch.cuda.device_count()
    if args.impl == "ours" and ndev < args.gpus:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "GB/s", "n_gpus": args.gpus,
                          "error": f"--gpus {args.gpus} but only {ndev} visible GPU(s); ranks never share a GPU"}),
              flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size-mib", type=int, default=128)
    ap.add_argument("--dtype", choices=["bf16", "f32"], default="bf16")
    ap.add_argument("--algo", choices=["auto", "recursive", "ring", "direct"], default="recursive",
                    help="configs[1] names recursive halving; auto = the library's measured selector")
    ap.add_argument("--retune", action="store_true", help="calibrate the selector on this box even if the table covers p")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-nccl-child", action="store_true")
    ap.add_argument("--nccl-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per launch, if measured")
    ap.add_argument("--profile", action="store_true", help="minimal launches for ncu: no soak/extra/e2e/cpu")
    args = ap.parse_args()
    if args.nccl_child:
        nccl_child(args)
        return
    if args.warmup < 3:
        args.warmup = 3
    if args.profile:
        args.no_extra = args.no_cpu = True
    ws = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":  # rank 0 alone runs on the host cores: no launcher needed
        run_reference(args)
        return
    if ws is None and args.gpus > 1:
        sys.exit(relaunch(args))
    if ws is not None and int(ws) != args.gpus and not (int(ws) == 1 and args.gpus == 1):
        print(json.dumps({"metric": METRIC, "value": None, "unit": "GB/s", "n_gpus": int(ws),
                          "error": f"WORLD_SIZE={ws} but --gpus {args.gpus}"}), flush=True)
        sys.exit(2)
    try:
        run_gpu(args)
    except Exception as exc:  # a failed run still leaves one parseable line (rank 0)
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": "GB/s",
                              "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
                              "warmup": args.warmup, "higher_is_better": True,
                              "error": f"{type(exc).__name__}: {exc}"[:400]}), flush=True)
        raise


if __name__ == "__main__":
    main()
