"""Worker of tests/test_gpu_sharded_device.py::test_device_protocol_two_processes (launched by
torch.distributed.run, 2 ranks on one GPU): row-sharded batches through the device-side
protocol (mpzch_sharded_*), each rank a PROCESS that maps the other's exchange region with CUDA
IPC -- the one-process-per-GPU deployment; gloo only carries the 128-byte records once."""
import os
import sys

import numpy as np


def workload(oracle):
    caps = [3000, 2500, 4000, 3500]
    P = 24
    uni = oracle.distinct_ids(73, 0, int(sum(caps) * 1.2))
    rng = np.random.default_rng(73)
    batches = []
    for b in range(6):
        n = 9000
        f = rng.integers(0, 3, n).astype(np.uint32) if b % 2 else None
        batches.append((uni[rng.integers(0, uni.size, n)], f, 1 + 25 * b))
    return caps, P, batches


def main():
    out = sys.argv[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch
    import torch.distributed as dist
    import pyoracle
    import paper_2602_17050_b200 as mz
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    caps, P, batches = workload(pyoracle)
    cfg = mz.TableConfig(caps, P, 7, 4, 3)
    rk = mz.ShardedRank(cfg, rank, world, 9000, device=0)
    recs = [None] * world
    dist.all_gather_object(recs, rk.export())
    rk.connect_ipc(recs)
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(40))
    for b, (ids, f, now) in enumerate(batches):
        sl = np.array_split(np.arange(ids.size), world)[rank]
        s, o, e = rk.process_batch(ids[sl], now, pol, None if f is None else f[sl])
        np.savez(os.path.join(out, f"r{rank}_b{b}.npz"), s=s, o=o, e=e, hw=rk.last_stats()["host_waits"])
    dist.barrier()  # no rank unmaps a peer region another rank may still be writing
    rk.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
