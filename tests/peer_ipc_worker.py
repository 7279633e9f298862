"""Worker of tests/test_gpu_sharded.py::test_peer_transport_two_processes (launched by
torch.distributed.run, 2 ranks on one GPU): row-sharded batches over the peer-memory transport
with CUDA IPC mappings; every rank saves its results for the test to check."""
import os
import sys

import numpy as np


def workload(oracle):
    caps = [3000, 2500, 4000, 3500]
    P = 24
    uni = oracle.distinct_ids(71, 0, int(sum(caps) * 1.2))
    rng = np.random.default_rng(71)
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
    from paper_2602_17050_b200.sharded import ShardedMpzchTable, TorchComm
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    caps, P, batches = workload(pyoracle)
    cfg = mz.TableConfig(caps, P, 7, 4, 3)
    st = ShardedMpzchTable(cfg, TorchComm(), device=0, transport="peer")
    pol = mz.EvictionPolicy.ttl(mz.TtlPolicy(40))
    for b, (ids, f, now) in enumerate(batches):
        sl = np.array_split(np.arange(ids.size), world)[rank]
        ti = torch.from_numpy(ids[sl].view(np.int64).copy()).cuda()
        tf = None if f is None else torch.from_numpy(f[sl].astype(np.int32)).cuda()
        s, o, e = st.process_batch(ti, now, pol, tf)
        np.savez(os.path.join(out, f"r{rank}_b{b}.npz"), s=s.cpu().numpy().view(np.uint64),
                 o=o.cpu().numpy(), e=e.cpu().numpy().view(np.uint64))
    st.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
