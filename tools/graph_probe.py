"""Real-mode CUDA graph capture probe: which kernels replay consistently."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

def main():
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"])); torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib
    comm = pkg.init_from_torch(device=dev.index); w = comm.world; L = _lib.lib()
    n = 4096
    gin = w.empty(n * p, torch.float32); gout = w.empty(n, torch.float32); gag = w.empty(n * p, torch.float32)
    gin.fill_(rank + 1)
    side = torch.cuda.Stream()
    rs = lambda s: L.pccl_reduce_scatter(comm.handle, 2, 0, gin.data_ptr(), gout.data_ptr(), n, 0, s)  # noqa
    ag = lambda s: L.pccl_all_gather(comm.handle, 0, gout.data_ptr(), gag.data_ptr(), n, 0, s)  # noqa
    agr = lambda s: L.pccl_all_gather(comm.handle, 1, gout.data_ptr(), gag.data_ptr(), n, 0, s)  # noqa
    rsd = lambda s: L.pccl_reduce_scatter(comm.handle, 0, 0, gin.data_ptr(), gout.data_ptr(), n, 0, s)  # noqa
    cases = {
        "rs_rec+ag_direct": lambda s: (rs(s), ag(s)),
        "rs_direct+rs_rec": lambda s: (rsd(s), rs(s)),
        "ag_direct+ag_ring": lambda s: (ag(s), agr(s)),
        "rs_rec+ag_ring": lambda s: (rs(s), agr(s)),
        "rs_rec_pull": lambda s: L.pccl_reduce_scatter(comm.handle, 2, 0, gin.data_ptr(), gout.data_ptr(), n, 0, s),
        "rs_direct_pull": lambda s: L.pccl_reduce_scatter(comm.handle, 0, 0, gin.data_ptr(), gout.data_ptr(), n, 0, s),
        "ag_direct_push": lambda s: L.pccl_all_gather(comm.handle, 0, gout.data_ptr(), gag.data_ptr(), n, 0, s),
        "ag_ring_push": lambda s: L.pccl_all_gather(comm.handle, 1, gout.data_ptr(), gag.data_ptr(), n, 0, s),
    }
    for pdl in (0,):
        w.set_param("pdl", pdl)
        for name, f in cases.items():
            for nodes in (1, 2):
                torch.cuda.synchronize(); dist.barrier()
                e0 = comm.epoch()
                f(side.cuda_stream); side.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    for _ in range(nodes):
                        f(side.cuda_stream)
                for _ in range(5):
                    g.replay()
                torch.cuda.synchronize()
                st = L.pccl_world_check(w.handle)
                e1 = comm.epoch()
                eps = [None] * p
                dist.all_gather_object(eps, (e1 - e0, st))
                if rank == 0:
                    print(f"pdl={pdl} {name:15s} nodes={nodes}: (epoch delta, status) per rank {eps}  expect {(1 + 5 * nodes) * (2 if '+' in name else 1)}", flush=True)
                if any(s for _, s in eps):
                    if rank == 0: print("  -> error, stopping"); 
                    dist.barrier(); dist.destroy_process_group(); return
    dist.destroy_process_group()

if __name__ == "__main__":
    main()
