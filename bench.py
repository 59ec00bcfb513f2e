"""Benchmark: reduce-scatter / all-gather bus bandwidth on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1]): reduce-scatter, bf16, 128 MiB
input per rank, recursive halving with the reduction fused into the peer-load
kernel. One *step* = one collective call. Metric: bus bandwidth
busbw = (S / t) * (p - 1) / p in GB/s (1e9 B/s), t = device time per call, max
over ranks.

* N = 1 (no torchrun): the reference's own shape, 8 *simulated* ranks
  (configs[0] "8 simulated ranks"), emulated on one B200: all eight ranks run
  in one cooperative launch of the same kernels, peer traffic is local HBM, so
  the roofline is HBM.
* N > 1 (torchrun, one process per GPU): p = N real ranks over CUDA-IPC peer
  memory on NVLink 5 / NVSwitch; roofline = NVLink. NCCL's
  reduce_scatter_tensor on the same bytes is timed beside it.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port of collkit's rechalf_reduce_scatter, ``oracle/``) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
PATTERN_CEILING_GBS = {"recursive": 642.0, "ring": 680.0, "direct": 634.0}  # profiles/r1_engine_probe_p4.md (rs ring pushes)
EMU_RANKS = 8


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


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
def cpu_reference(p: int, s_bytes: int, dtype: str, algo: str, steps: int, warmup: int):
    """Time the reference algorithm's CPU restatement on this host's cores:
    p simulated ranks, numpy, the per-step work of every rank in parallel
    threads (numpy releases the GIL in its kernels)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    from oracle import collectives as oc

    es = 2 if dtype == "bf16" else 4
    n = s_bytes // es // p
    rng = np.random.default_rng(0)
    ins = []
    for _ in range(p):
        x = rng.standard_normal(n * p).astype(np.float32)
        ins.append(oracle.f32_to_bf16(x) if dtype == "bf16" else x)
    # every host thread this process may use (affinity mask), capped so each
    # thread still gets >= 16 Ki elements of every chunk
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        threads = os.cpu_count() or 1
    threads = max(1, min(threads, n // 16384 or 1))
    pool = ThreadPoolExecutor(max_workers=threads)
    fn = oc.rechalf_reduce_scatter if algo == "recursive" else oc.ring_reduce_scatter

    def one_call():
        # the element range is split across threads (elementwise folds: every
        # element keeps its reduction order); numpy releases the GIL
        parts = threads
        bounds = np.linspace(0, n, parts + 1).astype(int)

        def run(i):
            lo, hi = bounds[i], bounds[i + 1]
            sub = [np.concatenate([x[c * n + lo : c * n + hi] for c in range(p)]) for x in ins]
            return fn(sub, dtype)

        list(pool.map(run, range(parts)))

    for _ in range(warmup):
        one_call()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        one_call()
        times.append(time.perf_counter() - t0)
    pool.shutdown()
    t = statistics.mean(times)
    return t, threads


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
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


def run_gpu(args):
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib
    from paper_2504_18658_b200.communicator import _emu_group, emulated_world

    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    real = world_size > 1
    # more ranks than GPUs (a functional check of the N-rank path on a smaller
    # box: ranks time-share GPUs, bootstrap over gloo, no NCCL / NVLS extras;
    # the numbers are not performance numbers)
    ndev = torch.cuda.device_count()
    # (a launcher that hands each rank its own GPU through CUDA_VISIBLE_DEVICES
    # shows exactly one device per process: that is not sharing)
    shared = real and world_size > ndev > 1
    if local_rank >= ndev:
        local_rank %= ndev
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    red_dev = torch.device("cpu") if shared else dev  # where max-over-ranks reductions live
    dist = None
    if real:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    p = world_size if real else EMU_RANKS
    S = args.size_mib << 20
    dtype = {"bf16": torch.bfloat16, "f32": torch.float32}[args.dtype]
    es = torch.empty(0, dtype=dtype).element_size()
    n = S // es // p
    code = _lib.DTYPES[args.dtype]
    stream = torch.cuda.current_stream(dev)
    L = _lib.lib()
    comm = pkg.init_from_torch(device=local_rank) if real else None
    # "auto": the library's measured selector; a GPU count the shipped table
    # does not cover is calibrated on this box first (collective, untimed)
    algo, selection = args.algo, "explicit (BASELINE configs[1]: recursive halving)" if args.algo == "recursive" \
        else "explicit"
    if algo == "auto":
        if real:
            from paper_2504_18658_b200 import selector, tuning

            if args.retune or not tuning.has_entries("reduce_scatter", p):
                tuned = tuning.autotune(comm, "reduce_scatter", S, dtype=dtype)
                selection = "autotuned on this box: " + ", ".join(f"{k} {v:.0f}" for k, v in tuned.items())
            else:
                selection = "measured selector table (data/flat_calibration.csv)"
            algo = selector.choose_algorithm("reduce_scatter", p, S)
        else:
            algo, selection = "recursive", "emulated N=1 headline: recursive halving"
    args.algo = algo
    a = _lib.ALGOS[algo]
    order = _lib.ORDERS["recursive" if algo == "recursive" else "ring"]

    # ---- symmetric buffers (inputs resident in HBM, zero-copy) ----
    if real:
        world = comm.world
        world.ensure_staging(int(L.pccl_staging_bytes(1, a, p, n, code)))
        sin = world.empty(n * p, dtype)
        sout = world.empty(n, dtype)
        sin.normal_()
        ghandle = comm.handle

        def call():
            _lib.check(L.pccl_reduce_scatter(ghandle, a, order, sin.data_ptr(), sout.data_ptr(), n, code,
                                             stream.cuda_stream))
    else:
        world = emulated_world(p, local_rank)
        group, _ = _emu_group(world, tuple(range(p)), 0)
        world.ensure_staging(int(L.pccl_staging_bytes(1, a, p, n, code)))
        sins = world.empty(n * p, dtype)
        souts = world.empty(n, dtype)
        for t in sins:
            t.normal_()
        sp = _lib.ptr_array([t.data_ptr() for t in sins])
        rp = _lib.ptr_array([t.data_ptr() for t in souts])

        def call():
            _lib.check(L.pccl_emu_reduce_scatter(group.handle, a, order, sp, rp, n, code, stream.cuda_stream))

    def barrier():
        torch.cuda.synchronize()
        if real:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- soak (for the clock sampler), warmup, timed region ----
    clocks = Clocks(local_rank)
    with clocks:
        # ~3 s of load for the clock sampler. The call count must be the same
        # on every rank (SPMD: each rank issues the same collectives), so it is
        # derived from a max-over-ranks estimate, never from local wall clock.
        if not args.profile:
            for _ in range(3):  # first launches load modules: keep them out of the estimate
                call()
            t_est = time_calls(call, 5, stream)
            if real:
                tt = torch.tensor([t_est], device=red_dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_est = float(tt.item())
            for i in range(max(20, min(60000, int(3.0 / max(t_est, 1e-6))))):
                call()
                if i % 50 == 49:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
        for _ in range(args.warmup):
            call()
        barrier()
        t_call = time_calls(call, args.steps, stream)
        world.check()
        barrier()
    if real:
        tt = torch.tensor([t_call], device=red_dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_call = float(tt.item())
    value = busbw(S, p, t_call)

    # ---- extras: the other algorithms / all-gather / NCCL, same bytes ----
    extra = {}
    if not args.no_extra:
        try:
            def measure(fn, k=max(5, args.steps)):
                for _ in range(3):
                    fn()
                barrier()
                t = time_calls(fn, k, stream)
                world.check()
                if real:
                    tt = torch.tensor([t], device=red_dev, dtype=torch.float64)
                    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                    t = float(tt.item())
                return t

            for alg2 in ("direct", "ring", "recursive"):
                a2 = _lib.ALGOS[alg2]
                o2 = _lib.ORDERS["recursive" if alg2 == "recursive" else "ring"]
                world.ensure_staging(int(L.pccl_staging_bytes(1, a2, p, n, code)))
                if real:
                    f = lambda: _lib.check(L.pccl_reduce_scatter(ghandle, a2, o2, sin.data_ptr(), sout.data_ptr(), n, code,  # noqa: E731
                                                                stream.cuda_stream))
                else:
                    f = lambda: _lib.check(L.pccl_emu_reduce_scatter(group.handle, a2, o2, sp, rp, n, code,  # noqa: E731
                                                                    stream.cuda_stream))
                t = measure(f)
                extra[f"rs_{args.dtype}_{args.size_mib}MiB_{alg2}"] = {"busbw_gbs": round(busbw(S, p, t), 1),
                                                                       "us": round(t * 1e6, 1)}
            # all-gather fp32 64 MiB output (configs[0] / C1 shape)
            S_ag = 64 << 20
            n_ag = S_ag // 4 // p
            if real:
                ag_in = world.empty(n_ag, torch.float32)
                ag_out = world.empty(n_ag * p, torch.float32)
                ag_in.normal_()
            else:
                ag_ins = world.empty(n_ag, torch.float32)
                ag_outs = world.empty(n_ag * p, torch.float32)
                agsp = _lib.ptr_array([t.data_ptr() for t in ag_ins])
                agrp = _lib.ptr_array([t.data_ptr() for t in ag_outs])
            for alg2 in ("direct", "ring", "recursive"):
                a2 = _lib.ALGOS[alg2]
                world.ensure_staging(int(L.pccl_staging_bytes(0, a2, p, n_ag, 0)))
                if real:
                    f = lambda: _lib.check(L.pccl_all_gather(ghandle, a2, ag_in.data_ptr(), ag_out.data_ptr(), n_ag, 0,  # noqa: E731
                                                            stream.cuda_stream))
                else:
                    f = lambda: _lib.check(L.pccl_emu_all_gather(group.handle, a2, agsp, agrp, n_ag, 0,  # noqa: E731
                                                                stream.cuda_stream))
                t = measure(f)
                extra[f"ag_f32_64MiB_{alg2}"] = {"busbw_gbs": round(busbw(S_ag, p, t), 1), "us": round(t * 1e6, 1)}
            if real and not shared:
                nin = torch.empty(n * p, dtype=dtype, device=dev).normal_()
                nout = torch.empty(n, dtype=dtype, device=dev)
                t = measure(lambda: dist.reduce_scatter_tensor(nout, nin))
                extra[f"nccl_rs_{args.dtype}_{args.size_mib}MiB"] = {"busbw_gbs": round(busbw(S, p, t), 1),
                                                                    "us": round(t * 1e6, 1),
                                                                    "nccl": ".".join(map(str, torch.cuda.nccl.version()))}
                agi = torch.empty(n_ag, dtype=torch.float32, device=dev).normal_()
                ago = torch.empty(n_ag * p, dtype=torch.float32, device=dev)
                t = measure(lambda: dist.all_gather_into_tensor(ago, agi))
                extra["nccl_ag_f32_64MiB"] = {"busbw_gbs": round(busbw(S_ag, p, t), 1), "us": round(t * 1e6, 1)}
                del nin, nout, agi, ago

            # the metric's range (64-256 MB): both collectives, every flat algorithm, at its ends
            for S_r in (64 << 20, 256 << 20):
                for coll, dt_r in (("ag", torch.float32), ("rs", torch.bfloat16)):
                    es_r = torch.empty(0, dtype=dt_r).element_size()
                    n_r = S_r // es_r // p
                    code_r = _lib.DTYPES["f32" if dt_r == torch.float32 else "bf16"]
                    c_in, c_out = (n_r, n_r * p) if coll == "ag" else (n_r * p, n_r)
                    if real:
                        r_in, r_out = world.empty(c_in, dt_r), world.empty(c_out, dt_r)
                        r_in.normal_()
                    else:
                        r_ins, r_outs = world.empty(c_in, dt_r), world.empty(c_out, dt_r)
                        for t_ in r_ins:
                            t_.normal_()
                        r_sp = _lib.ptr_array([t_.data_ptr() for t_ in r_ins])
                        r_rp = _lib.ptr_array([t_.data_ptr() for t_ in r_outs])
                    for alg2 in ("direct", "ring", "recursive"):
                        a2 = _lib.ALGOS[alg2]
                        o2 = _lib.ORDERS["recursive" if alg2 == "recursive" else "ring"]
                        world.ensure_staging(int(L.pccl_staging_bytes(0 if coll == "ag" else 1, a2, p, n_r, code_r)))
                        if coll == "ag" and real:
                            f = lambda: _lib.check(L.pccl_all_gather(ghandle, a2, r_in.data_ptr(), r_out.data_ptr(),  # noqa: E731
                                                                    n_r, code_r, stream.cuda_stream))
                        elif coll == "ag":
                            f = lambda: _lib.check(L.pccl_emu_all_gather(group.handle, a2, r_sp, r_rp, n_r, code_r,  # noqa: E731
                                                                        stream.cuda_stream))
                        elif real:
                            f = lambda: _lib.check(L.pccl_reduce_scatter(ghandle, a2, o2, r_in.data_ptr(),  # noqa: E731
                                                                        r_out.data_ptr(), n_r, code_r, stream.cuda_stream))
                        else:
                            f = lambda: _lib.check(L.pccl_emu_reduce_scatter(group.handle, a2, o2, r_sp, r_rp, n_r,  # noqa: E731
                                                                            code_r, stream.cuda_stream))
                        t = measure(f)
                        tag = f"{coll}_{'f32' if coll == 'ag' else 'bf16'}_{S_r >> 20}MiB_{alg2}"
                        extra[tag] = {"busbw_gbs": round(busbw(S_r, p, t), 1), "us": round(t * 1e6, 1)}
                    if real:
                        del r_in, r_out
                    else:
                        del r_ins, r_outs

            # NVLS: switch multicast stores (AG) / switch reductions (bf16 RS)
            nvls_ok = real and not shared
            if nvls_ok:
                from paper_2504_18658_b200 import nvls as NV

                try:
                    nvls_ok = NV.nvls_supported(world)
                except Exception as exc:  # noqa: BLE001 - optional path, never costs the rest
                    extra["nvls_error"] = f"{type(exc).__name__}: {exc}"[:200]
                    nvls_ok = False
            if nvls_ok:
                try:
                    P7n = 12 * 4096 * 4096 + 13 * 4096
                    seg = NV.create_nvls_segment(world, max(S, P7n * 2 + 4096))
                    try:
                        nx = seg.tensor(0, n * p, torch.bfloat16)
                        nx.normal_()
                        ny = torch.empty(n, dtype=torch.bfloat16, device=dev)
                        t = measure(lambda: NV.nvls_reduce_scatter(comm, seg, nx, ny))
                        extra[f"nvls_rs_bf16_{args.size_mib}MiB"] = {"busbw_gbs": round(busbw(S, p, t), 1),
                                                                   "us": round(t * 1e6, 1)}
                        for S_a, dt_a, nm in ((64 << 20, torch.float32, "ag_f32_64MiB"),
                                              (P7n // p * p * 2, torch.bfloat16, "fsdp7b_layer_ag_bf16")):
                            n_a = S_a // torch.empty(0, dtype=dt_a).element_size() // p
                            ax = torch.empty(n_a, dtype=dt_a, device=dev).normal_()
                            ay = seg.tensor(0, n_a * p, dt_a)
                            t = measure(lambda: NV.nvls_all_gather(comm, seg, ax, ay))
                            extra[f"nvls_{nm}"] = {"busbw_gbs": round(busbw(S_a, p, t), 1), "us": round(t * 1e6, 1)}
                        n7 = P7n // p
                        gx = seg.tensor(0, n7 * p, torch.bfloat16)
                        gx.normal_()
                        gy = torch.empty(n7, dtype=torch.bfloat16, device=dev)
                        t = measure(lambda: NV.nvls_reduce_scatter(comm, seg, gx, gy))
                        extra["nvls_fsdp7b_layer_rs_bf16"] = {"busbw_gbs": round(busbw(n7 * p * 2, p, t), 1),
                                                              "us": round(t * 1e6, 1)}
                    finally:
                        seg.close()
                except Exception as exc:  # noqa: BLE001 - optional path, never costs the rest
                    extra["nvls_error"] = f"{type(exc).__name__}: {exc}"[:200]
                    world.check()  # a device error (poisoned world) still ends the extras

            # C3: hierarchical AG + RS, 256 MiB, virtual N x M groupings
            S_h = 256 << 20
            grids = [(N, p // N) for N in (2, 4) if p % N == 0 and 1 < N < p]
            if grids:
                n_h = S_h // 4 // p
                if real:
                    h_ag_in, h_ag_out = world.empty(n_h, torch.float32), world.empty(n_h * p, torch.float32)
                    h_rs_in, h_rs_out = world.empty(n_h * p, torch.float32), world.empty(n_h, torch.float32)
                    h_ag_in.normal_()
                    h_rs_in.normal_()
                else:
                    hai, hao = world.empty(n_h, torch.float32), world.empty(n_h * p, torch.float32)
                    hri, hro = world.empty(n_h * p, torch.float32), world.empty(n_h, torch.float32)
                    ptrs = {k: _lib.ptr_array([t.data_ptr() for t in v]) for k, v in
                            dict(ai=hai, ao=hao, ri=hri, ro=hro).items()}
                world.ensure_staging(int(L.pccl_staging_bytes(1, 3, p, n_h, 0)))
                for (N, M) in grids:
                    inter = "recursive" if N >= 4 else "ring"
                    ia = _lib.ALGOS[inter]
                    if real:
                        fa = lambda: _lib.check(L.pccl_hier_all_gather(world.handle, N, M, ia, h_ag_in.data_ptr(),  # noqa: E731
                                                                      h_ag_out.data_ptr(), n_h, 0, stream.cuda_stream))
                        fr = lambda: _lib.check(L.pccl_hier_reduce_scatter(world.handle, N, M, ia, h_rs_in.data_ptr(),  # noqa: E731
                                                                          h_rs_out.data_ptr(), n_h, 0, stream.cuda_stream))
                    else:
                        fa = lambda: _lib.check(L.pccl_emu_hier_all_gather(world.handle, N, M, ia, ptrs["ai"], ptrs["ao"],  # noqa: E731
                                                                          n_h, 0, stream.cuda_stream))
                        fr = lambda: _lib.check(L.pccl_emu_hier_reduce_scatter(world.handle, N, M, ia, ptrs["ri"],  # noqa: E731
                                                                              ptrs["ro"], n_h, 0, stream.cuda_stream))
                    for nm, f in (("ag", fa), ("rs", fr)):
                        t = measure(f)
                        extra[f"hier_{nm}_f32_256MiB_{N}x{M}_{inter}"] = {"busbw_gbs": round(busbw(S_h, p, t), 1),
                                                                          "us": round(t * 1e6, 1)}

            # C5: FSDP / ZeRO-3 GPT-3-style 7B per-layer shapes (12h^2 + 13h params, h = 4096), bf16
            if real:
                P7 = 12 * 4096 * 4096 + 13 * 4096
                n7 = P7 // p
                S7 = n7 * p * 2
                prm = world.empty(n7, torch.bfloat16)
                full = world.empty(n7 * p, torch.bfloat16)
                grad = world.empty(n7 * p, torch.bfloat16)
                gsh = world.empty(n7, torch.bfloat16)
                prm.normal_()
                grad.normal_()
                world.ensure_staging(int(L.pccl_staging_bytes(1, 2, p, n7, 1)))
                t = measure(lambda: pkg.all_gather_into_tensor(full, prm, comm))
                extra["fsdp7b_layer_ag_bf16"] = {"busbw_gbs": round(busbw(S7, p, t), 1), "us": round(t * 1e6, 1),
                                                 "bytes_out": S7, "algorithm": pkg.choose_algorithm("all_gather", p, S7)}
                t = measure(lambda: pkg.reduce_scatter_tensor(gsh, grad, comm))
                extra["fsdp7b_layer_rs_bf16"] = {"busbw_gbs": round(busbw(S7, p, t), 1), "us": round(t * 1e6, 1),
                                                 "bytes_in": S7, "algorithm": pkg.choose_algorithm("reduce_scatter", p, S7)}
                if not shared:
                    nfull = torch.empty(n7 * p, dtype=torch.bfloat16, device=dev)
                    nprm = torch.empty(n7, dtype=torch.bfloat16, device=dev).normal_()
                    t = measure(lambda: dist.all_gather_into_tensor(nfull, nprm))
                    extra["nccl_fsdp7b_layer_ag_bf16"] = {"busbw_gbs": round(busbw(S7, p, t), 1),
                                                          "us": round(t * 1e6, 1)}
                    ngrad = torch.empty(n7 * p, dtype=torch.bfloat16, device=dev).normal_()
                    t = measure(lambda: dist.reduce_scatter_tensor(nprm, ngrad))
                    extra["nccl_fsdp7b_layer_rs_bf16"] = {"busbw_gbs": round(busbw(S7, p, t), 1),
                                                          "us": round(t * 1e6, 1)}
                    del nfull, nprm, ngrad
        except Exception as exc:  # an extra must never cost the headline line
            extra["error"] = f"{type(exc).__name__}: {exc}"[:300]
            if rank == 0:
                print(f"[bench] extra measurements aborted: {exc!r}", file=sys.stderr, flush=True)

    # ---- e2e through the public API with host buffers ----
    if args.profile:
        e2e = None
    elif "error" in extra:  # a device error poisons the world: no further collectives
        e2e = {"value": None, "unit": "GB/s", "error": "skipped after: " + extra["error"][:200]}
    else:
        e2e = run_e2e(args, pkg, real, p, S, dtype, dev, comm if real else None, dist)

    # ---- roofline of the dominant kernel (the measured call itself) ----
    pk, src = peaks()
    if real:
        achieved = value  # algorithmic NVLink bytes per GPU per launch / launch time
        roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_MEASURED_GBS,
                "unit": "GB/s", "frac": round(achieved / NVLINK_MEASURED_GBS, 4),
                "frac_of_nominal_900": round(achieved / NVLINK_NOMINAL_GBS, 4),
                # the traffic pattern's own measured ceiling (raw 16-byte loops, no flags, p=4,
                # tools/probe.py / profiles/r1_engine_probe_p4.md): recursive halving and ring are
                # pairwise bidirectional peer loads, direct is all-to-all peer loads
                "pattern_ceiling": {"gbs": PATTERN_CEILING_GBS.get(algo), "frac": round(
                    achieved / PATTERN_CEILING_GBS[algo], 4) if algo in PATTERN_CEILING_GBS else None,
                    "source": "tools/probe.py raw loops at p=4: recursive = bidirectional LDG pull, ring = "
                              "bidirectional STG push, direct = all-to-all LDG pull"},
                "peak_source": "B200_PROFILING.md measured peer copy (nominal 900)",
                "algorithmic_bytes_per_launch": int(S * (p - 1) / p), "traffic": None}
    else:
        hbm = rs_algorithmic_hbm_bytes(algo, p, n * es)
        achieved = hbm / t_call / 1e9
        peak = float(pk.get("hbm_gbs", 6650.0))
        traffic = args.traffic
        if traffic is None and algo == "recursive" and args.dtype == "bf16" and args.size_mib == 128:
            # dram__bytes_read.sum + dram__bytes_write.sum of this launch, ncu --set full
            # (profiles/r1_ncu_k_rs_rec_emulated.md, r1c): 1.878951 GB + 0.916030 GB
            traffic = 2794981208
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                "algorithmic_bytes_per_launch": hbm, "traffic": traffic,
                "traffic_source": "ncu --set full capture, profiles/r1_ncu_k_rs_rec_emulated.md" if traffic else None}

    cpu = None
    if rank == 0 and not real and not args.no_cpu:
        s_cpu = 16 << 20
        t_cpu, cores = cpu_reference(p, s_cpu, args.dtype, algo, steps=3, warmup=1)
        cpu = {"value": round(busbw(s_cpu, p, t_cpu), 4), "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": f"oracle rechalf_reduce_scatter {args.dtype}, p={p} ranks, S=16 MiB/rank, 3 calls "
                         f"(numpy, {cores} threads)"}

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
            "data": "synthetic (standard normal, resident in symmetric HBM segments)"
                    + ("; SHARED GPUS (more ranks than GPUs): functional check, not a performance number" if shared
                       else ""),
            "config": {
                "workload": (f"reduce-scatter {args.dtype}, {args.size_mib} MiB input/rank, {algo} "
                             f"(fused reduction), p={p} " + ("GPUs over NVLink/NVSwitch" if real else
                                                             "simulated ranks emulated on 1 B200 (HBM-bound)")),
                "collective": "reduce_scatter",
                "algorithm": algo,
                "selection": selection,
                "p": p,
                "S_bytes": S,
                "parallelism": f"dp{p}" if real else "emulated-8-ranks-1gpu",
                "l2": "inputs larger than L2 (per-rank input 128 MiB > 126 MB L2)",
                "ctas_per_rank": int(os.environ.get("PCCL_CTAS", "0")) or "auto",
            },
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": clocks.summary(),
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if real:
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
            y = fn(comm, x)
            per.append(time.perf_counter() - t0)
        tt = torch.tensor(per, device="cpu" if dist.get_backend() == "gloo" else dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)  # per step: the slowest rank
        per = tt.tolist()
        h2d, d2h = n * p * es * p, n * es * p
    else:
        xs = [torch.empty(n * p, dtype=dtype).normal_().pin_memory() for _ in range(p)]
        timing = {}

        def body(c):
            for _ in range(2):
                fn(c, xs[c.rank])
            per = []
            for _ in range(steps):
                t0 = time.perf_counter()
                y = fn(c, xs[c.rank])
                per.append(time.perf_counter() - t0)
            if c.rank == 0:  # the emulated ranks finish each step together (one launch)
                timing["per"] = per
            return None

        pkg.run_ranks(p, body, device=dev.index)
        per = timing["per"]
        h2d, d2h = n * p * es * p, n * es * p
    # host-link-bound and noisy on shared hosts (single steps up to 2x the
    # typical one): the value is the median step, the mean is reported beside it
    dt = statistics.median(per)
    mean = sum(per) / len(per)
    return {"value": round(busbw(S, p, dt), 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(dt * 1e3, 3),
            "ms_per_step_mean": round(mean * 1e3, 3), "steps": len(per), "statistic": "median step",
            "path": f"paper_2504_18658_b200.{fn.__name__}(comm, pinned host tensor) -> host tensor "
                    "(sliced, copies overlapped with the collective)"}


def run_reference(args):
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p = world_size if world_size > 1 else EMU_RANKS
    if args.algo in ("auto", "direct"):  # the reference has ring and recursive halving only
        args.algo = "recursive"
    s_sample = 16 << 20
    t, cores = cpu_reference(p, s_sample, args.dtype, args.algo, steps=args.steps, warmup=args.warmup)
    v = busbw(s_sample, p, t)
    sample = (f"oracle port of collkit {args.algo} reduce-scatter ({args.dtype}), p={p} simulated ranks, "
              f"16 MiB/rank sample of the {args.size_mib} MiB workload, numpy on {cores} host threads")
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": world_size, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": f"reduce-scatter {args.dtype}, {args.size_mib} MiB input/rank, {args.algo}, p={p}",
                   "collective": "reduce_scatter", "algorithm": args.algo, "p": p},
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per launch, if measured")
    ap.add_argument("--profile", action="store_true", help="minimal launches for ncu: no soak/extra/e2e/cpu")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.profile:
        args.no_extra = args.no_cpu = True
    if args.impl == "reference":
        run_reference(args)
        return
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
