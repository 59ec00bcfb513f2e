"""Memory-model stress for the pull kernels' publish.

Pull kernels publish data that lives in the writer's own HBM. With
local_fence = 1 (default) the signal is `fence.acq_rel.gpu` + `st.relaxed.sys`
(the writer's L2 is the point of coherence every NVLink reader goes through);
local_fence = 0 uses `st.release.sys`. This runs N back-to-back collectives
per configuration with the INPUTS REWRITTEN BY A KERNEL RIGHT BEFORE EVERY
CALL (value base + i at iteration i) and a random per-rank launch skew, and
checks every output on the device (integer-valued data: exact in any
order), so a reader that saw a flag before the data would read iteration
i-1's values and be counted.

    torchrun --nproc-per-node 4 tools/litmus.py --iters 100000
"""
import argparse
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100000, help="collectives per (local_fence) setting")
    ap.add_argument("--fences", default="1,0")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--movement", choices=["pull", "default", "ll128"], default="pull",
                    help="pull: force pull kernels (the local_fence publish); default: the library's choice")
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib

    L = _lib.lib()
    comm = pkg.init_from_torch(device=dev.index)
    w = comm.world
    w.set_param("ll_max", 0)        # flag protocol only (LL carries its flags inside the data)
    if a.movement == "pull":
        w.set_param("rs_variant", 0)    # pull
        w.set_param("ag_variant", 0)    # pull
    if a.movement != "ll128":
        w.set_param("ll128_max", 0)     # flag protocol only
    if a.movement == "ll128":
        w.set_param("ag_variant", 8)    # LL128 line protocol for every direct collective that fits a region
        w.set_param("rs_variant", 8)
    # "default": the library's choice for symmetric buffers (RS pull, AG push
    # with the rank-level final publish)
    stream = torch.cuda.current_stream(dev).cuda_stream
    pow2 = p & (p - 1) == 0
    algos = ["direct", "ring"] + (["recursive"] if pow2 else [])
    sizes = [64 << 10, 256 << 10, 1 << 20, 4 << 20]  # bytes per rank: RS input / AG output
    bufs = {}
    for S in sizes:
        n = S // 4 // p
        g = torch.Generator(device=dev).manual_seed(1000 + rank)
        base_rs = torch.randint(-50, 51, (n * p,), generator=g, device=dev).float()
        base_ag = torch.randint(-50, 51, (n,), generator=g, device=dev).float()
        all_rs = [torch.empty_like(base_rs) for _ in range(p)]
        dist.all_gather(all_rs, base_rs)
        all_ag = [torch.empty_like(base_ag) for _ in range(p)]
        dist.all_gather(all_ag, base_ag)
        bufs[S] = dict(n=n, base_rs=base_rs, base_ag=base_ag,
                       want_rs=sum(all_rs)[rank * n:(rank + 1) * n].clone(), want_ag=torch.cat(all_ag),
                       x=w.empty(n * p, torch.float32), y=w.empty(n, torch.float32),
                       ax=w.empty(n, torch.float32), ay=w.empty(n * p, torch.float32))
        w.ensure_staging(int(L.pccl_staging_bytes(1, 2, p, n, 0)))
    err = torch.zeros((), dtype=torch.int64, device=dev)
    rng = random.Random(a.seed)          # same sequence on every rank (SPMD)
    skew = random.Random(a.seed * 7919 + rank)  # per-rank launch skew
    report = []
    for fence in map(int, a.fences.split(",")):
        w.set_param("local_fence", fence)
        torch.cuda.synchronize()
        dist.barrier()
        err.zero_()
        t0 = time.time()
        counts = {}
        for i in range(a.iters):
            S = rng.choice(sizes)
            algo = rng.choice(algos)
            coll = rng.choice(["rs", "ag"])
            b = bufs[S]
            n = b["n"]
            it = float(i % 1000)
            if skew.random() < 0.2:
                torch.cuda._sleep(skew.randint(100, 20000))  # ~0.05-10 us of skew on this rank
            if coll == "rs":
                torch.add(b["base_rs"], it, out=b["x"])  # inputs written right before the call
                o = _lib.ORDERS["recursive" if algo == "recursive" else "ring"]
                _lib.check(L.pccl_reduce_scatter(comm.handle, _lib.ALGOS[algo], o, b["x"].data_ptr(),
                                                 b["y"].data_ptr(), n, 0, stream))
                err += (b["y"] != b["want_rs"] + p * it).sum()
            else:
                torch.add(b["base_ag"], it, out=b["ax"])
                _lib.check(L.pccl_all_gather(comm.handle, _lib.ALGOS[algo], b["ax"].data_ptr(), b["ay"].data_ptr(),
                                             n, 0, stream))
                err += (b["ay"] != b["want_ag"] + it).sum()
            counts[(coll, algo)] = counts.get((coll, algo), 0) + 1
            if i % 2000 == 1999:
                torch.cuda.synchronize()
                w.check()
        torch.cuda.synchronize()
        w.check()
        dt = time.time() - t0
        tot = torch.tensor([int(err)], device=dev)
        dist.all_reduce(tot)
        report.append(f"local_fence={fence}: {a.iters} calls per rank in {dt:.1f} s, mismatched elements "
                      f"(all ranks) = {int(tot)}; mix " + ", ".join(f"{k[0]}/{k[1]} {v}" for k, v in sorted(counts.items())))
    if rank == 0:
        print(f"== litmus p={p} sizes {[s >> 10 for s in sizes]} KiB, {a.movement} data movement, flag protocol", flush=True)
        for r in report:
            print("  " + r, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
