"""Sweep CTAs-per-rank / sub-slices for every algorithm (real mode, torchrun).

    torchrun --nproc-per-node N tools/tune.py [--size-mib 128] [--ctas 16,32,64] [--nsub 1,2,4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size-mib", type=int, default=128)
    ap.add_argument("--ctas", default="16,32,64,96,128")
    ap.add_argument("--nsub", default="1")
    ap.add_argument("--threads", default="512")
    ap.add_argument("--colls", default="ag_f32,rs_bf16")
    ap.add_argument("--algos", default="direct,ring,recursive")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--variants", default="-1")
    ap.add_argument("--tma", default="4x32768", help="stages x tile bytes list, comma separated")
    ap.add_argument("--items", default="0", help="item_kib list (direct kernels; 0 = static CTA slices)")
    ap.add_argument("--params", default="", help="key=value,... world params applied first")
    args = ap.parse_args()
    rank = int(os.environ["RANK"])
    p = int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib

    L = _lib.lib()
    comm = pkg.init_from_torch(device=dev.index)
    world = comm.world
    for kv in filter(None, args.params.split(",")):
        k, v = kv.split("=")
        world.set_param(k, int(v))
    S = args.size_mib << 20
    stream = torch.cuda.current_stream(dev)
    results = []
    for coll in args.colls.split(","):
        kind, dt = coll.split("_")
        dtype = torch.bfloat16 if dt == "bf16" else torch.float32
        es = 2 if dt == "bf16" else 4
        code = _lib.DTYPES[dt]
        n = S // es // p
        if kind == "ag":
            sin = world.empty(n, dtype)
            sout = world.empty(n * p, dtype)
        else:
            sin = world.empty(n * p, dtype)
            sout = world.empty(n, dtype)
        sin.normal_()
        for algo in args.algos.split(","):
            if algo == "recursive" and p & (p - 1):
                continue
            a = _lib.ALGOS[algo]
            world.ensure_staging(int(L.pccl_staging_bytes(0 if kind == "ag" else 1, a, p, n, code)))
            combos = []
            for v in map(int, args.variants.split(",")):
                if v in (2, 3, 4) and algo != "direct":
                    continue
                if v in (2, 3) and kind == "rs":
                    continue
                if v == 5 and kind == "ag" and algo == "direct":  # AG 5: copy engine (ring / recursive doubling)
                    continue
                if v == 5 and kind == "rs" and algo != "direct":  # RS 5: pipelined push (direct)
                    continue
                for tm in (args.tma.split(",") if v >= 2 else ["0x0"]):
                    combos.append((v, *map(int, tm.split("x"))))
            for (variant, stg, tile) in combos:
              world.set_param("ag_variant" if kind == "ag" else "rs_variant", variant)
              if stg:
                  world.set_param("tma_stages", stg)
                  world.set_param("tma_tile", tile)
              for thr, ctas in [(th, ct) for th in map(int, args.threads.split(",")) for ct in map(int, args.ctas.split(","))]:
                world.set_param("threads", thr)
                for nsub, item in [(ns, it) for ns in map(int, args.nsub.split(",")) for it in map(int, args.items.split(","))]:
                    if item != int(args.items.split(",")[0]) and algo != "direct":
                        continue
                    world.set_tuning(ctas, nsub)
                    world.set_param("item_kib", item)
                    if kind == "ag":
                        f = lambda: _lib.check(L.pccl_all_gather(comm.handle, a, sin.data_ptr(), sout.data_ptr(), n,  # noqa
                                                                code, stream.cuda_stream))
                    else:
                        o = _lib.ORDERS["recursive" if algo == "recursive" else "ring"]
                        f = lambda: _lib.check(L.pccl_reduce_scatter(comm.handle, a, o, sin.data_ptr(),  # noqa
                                                                    sout.data_ptr(), n, code, stream.cuda_stream))
                    for _ in range(3):
                        f()
                    torch.cuda.synchronize()
                    dist.barrier()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(args.iters):
                        f()
                    e1.record()
                    torch.cuda.synchronize()
                    world.check()
                    t = torch.tensor([e0.elapsed_time(e1) / args.iters], device=dev)
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    us = float(t) * 1e3
                    bw = S * (p - 1) / p / (us * 1e-6) / 1e9
                    results.append(dict(coll=coll, algo=algo, variant=variant, stages=stg, tile=tile, ctas=ctas, threads=thr,
                                        nsub=nsub, item_kib=item, us=round(us, 1), busbw=round(bw, 1)))
                    if rank == 0:
                        print(f"p={p} {coll:8s} {algo:9s} v={variant} tma={stg}x{tile:6d} thr={thr:3d} ctas={ctas:4d} nsub={nsub:2d} "
                              f"item={item:3d} {us:9.1f} us {bw:7.1f} GB/s", flush=True)
              world.set_param("ag_variant", -1)
              world.set_param("rs_variant", -1)
    # NCCL reference points
    for coll in args.colls.split(","):
        kind, dt = coll.split("_")
        dtype = torch.bfloat16 if dt == "bf16" else torch.float32
        es = 2 if dt == "bf16" else 4
        n = S // es // p
        if kind == "ag":
            i = torch.randn(n, device=dev).to(dtype)
            o = torch.empty(n * p, device=dev, dtype=dtype)
            f = lambda: dist.all_gather_into_tensor(o, i)  # noqa
        else:
            i = torch.randn(n * p, device=dev).to(dtype)
            o = torch.empty(n, device=dev, dtype=dtype)
            f = lambda: dist.reduce_scatter_tensor(o, i)  # noqa
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = float(t) * 1e3
        bw = S * (p - 1) / p / (us * 1e-6) / 1e9
        if rank == 0:
            print(f"p={p} {coll:8s} NCCL      {us:9.1f} us {bw:7.1f} GB/s", flush=True)
        results.append(dict(coll=coll, algo="nccl", us=round(us, 1), busbw=round(bw, 1)))
    if rank == 0:
        os.makedirs("gpurun_out", exist_ok=True)
        with open(f"gpurun_out/tune_p{p}_{args.size_mib}MiB.json", "w") as fh:
            json.dump(results, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
