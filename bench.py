#!/usr/bin/env python
"""bench.py -- device-timed remapped IDs/s of the MPZCH batched remap path on B200.

Workload (the north star's headline): a 1B-slot table (2^30 rows, S=8
logical shards, max_probe=128, seed 7, eviction Disabled) prefilled through the API to
load 0.8 with DistinctIdStream(5)[0, N_pre), then batches of 4,194,304 positions:
90% uniform over the prefilled ids, 10% fresh ids (N_pre + k).  A step = one
process_batch over one batch.  IDs/s counts input positions (duplicates included, as
run_latency_bench does, proj/src/experiments.cpp:325,347).

  value     device-resident inputs, CUDA events on the launch stream, K steps
  e2e       the host-buffer C-ABI call (mpzch_process_batch) from pinned host memory:
            H2D ids + D2H slots/outcomes inside the timed region
  roofline  the probe kernel (dominant): algorithmic bytes (32-byte sectors it must read
            + per-position I/O) / its CUDA-event launch time, vs MEASURED_PEAKS hbm_gbs
  cpu_baseline / --impl reference
            the REFERENCE library (oracle/_ref, /root/reference/proj/src compiled by
            oracle/Makefile, OpenMP over all host cores) on the SAME workload: the 2^30-row
            layout, the same prefill and the same batch stream, each batch timed with
            steady_clock around process_batch alone (proj/src/experiments.cpp:339-347);
            cpu_baseline times 3 of those batches, --impl reference K of them.

Multi-GPU (torchrun, N>1): the same 1B-slot table row-sharded over the N ranks (each holds
8/N logical shards), every 4M-position batch split into N slices -- strong scaling of the fixed
C5 workload.  Default MPZCH_TRANSPORT=device: the device-side protocol of csrc/sharded.cu (ids to
owners and results back by stores into the other ranks' CUDA-IPC-mapped exchange regions over
NVLink, system-scope flags between the phases, every phase on the stream, one host wait per
batch, batches pipelined by ticket); MPZCH_TRANSPORT=peer|collective run the host-driven
protocol of paper_2602_17050_b200/sharded.py (peer stores or the NCCL all-to-all).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GOLD = -7046029254386353131          # 0x9E3779B97F4A7C15 as int64
M1 = -49064778989728563              # 0xff51afd7ed558ccd
M2 = -4265267296055464877            # 0xc4ceb9fe1a85ec53
S1 = -4658895280553007687            # 0xBF58476D1CE4E5B9
S2 = -7723592293110705685            # 0x94D049BB133111EB
LOW31 = (1 << 31) - 1


def _i64(v):
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def mix64_t(x, seed: int):
    """ids.hpp:35-43 on int64 tensors (wrapping multiply; logical shifts via masks)."""
    x = x ^ _i64(seed)
    x = x ^ ((x >> 33) & ((1 << 31) - 1))
    x = x * M1
    x = x ^ ((x >> 33) & ((1 << 31) - 1))
    x = x * M2
    return x ^ ((x >> 33) & ((1 << 31) - 1))


def distinct_ids_t(seed: int, idx):
    """DistinctIdStream::at, rng.hpp:40-50, on an int64 index tensor."""
    left = (idx >> 31) & LOW31
    right = idx & LOW31
    for r in range(4):
        f = mix64_t(right | (r << 32), seed) & LOW31
        left, right = right, left ^ f
    return (left << 31) | right


def splitmix_t(seed: int, k):
    """k-th (0-based) output of SplitMix64(seed), rng.hpp:15-21."""
    z = (k + 1) * GOLD + _i64(seed)
    z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * S1
    z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * S2
    return z ^ ((z >> 31) & ((1 << 33) - 1))


def batch_indices(torch, device, pool: int, batch: int, b: int, fresh_base: int, seed: int,
                  fresh_pct: int = 10):
    """Stream index of each position of batch b: with probability fresh_pct% a fresh index
    (pool + running count), else uniform over [0, pool).  Two SplitMix64 draws per position
    (coin, pick); returns (indices, fresh count)."""
    k = torch.arange(2 * batch * b, 2 * batch * (b + 1), dtype=torch.int64, device=device)
    d = splitmix_t(seed, k) & ((1 << 63) - 1)
    coin = d[0::2] % 100
    pick = d[1::2] % pool
    fresh = coin < fresh_pct
    rank = torch.cumsum(fresh.to(torch.int64), 0) - 1
    idx = torch.where(fresh, fresh_base + rank, pick)
    return idx, int(fresh.sum().item())


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []      # (t, fields)
        self.windows = []   # load windows (t0, t1)
        self.proc = None

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)

    def under_load(self):
        return [r for (t, r) in self.rows if any(a <= t <= b for a, b in self.windows)]

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.under_load()
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples_under_load": len(rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def random_sector_ceiling():
    """Measured uniform-random 32-byte read ceiling (tools/sector_bench.cu), GB/s of useful bytes."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "sector_ceiling_r*.json")))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        return max(r["useful_gbs"] for r in d["results"] if r["op"] == "read" and r["bytes"] == 32)
    except Exception:
        return None


def random_access_ceiling():
    """Measured random DRAM access rate (tools/sector_probe.cu): G accesses/s over a 16 GiB
    array for 32-byte reads -- the same rate holds for 128-byte line reads -- and for 8-byte
    writes (profiles/line_ceiling_r01.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "line_ceiling_r01.json")))
        t = [r for r in d["timings"] if r.get("gib") == 16]
        rd = max(r.get("G_sectors_s", r.get("G_accesses_s", 0)) for r in t if r["kernel"].startswith("cg_"))
        w8 = max(r["G_sectors_s"] for r in t if r["kernel"] == "write8")
        return {"read_g_per_s": rd, "write8_g_per_s": w8}
    except Exception:
        return None


def probe_dram_accesses():
    """Random DRAM accesses per k_probe launch from the committed ncu capture: 128-byte line
    fetches (read sectors / 4: the L2 fetches whole lines for random reads) + written sectors."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_probe_summary.json")))
        return d["dram_read_bytes"] / 128.0 + d["dram_write_bytes"] / 32.0
    except Exception:
        return None


def independent_ceiling(probe_ms):
    """k_probe against the random-access ceiling measured with PyTorch's OWN gather / scatter
    kernels (profiles/random_ceiling_torch_r02.json: index_select / index_put_ of 8-byte rows at
    random over a 16 GiB array -- independent of this repo's code): the launch's DRAM reads
    (128-byte line fetches) at the read rate plus its written sectors at the write rate, done one
    after the other, is the time the memory system needs for that access mix; frac > 1 means the
    reads and writes overlapped."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "random_ceiling_torch_r02.json")))
        rows = [r for r in d["rows"] if r["gib"] == 16]
        rd = next(r["G_accesses_s"] for r in rows if r["op"] == "index_select 8 B rows")
        wr = next(r["G_accesses_s"] for r in rows if r["op"] == "index_put_ 8 B rows")
        p = json.load(open(os.path.join(ROOT, "profiles", "ncu_probe_summary.json")))
        reads, writes = p["dram_read_bytes"] / 128.0, p["dram_write_bytes"] / 32.0
        ceil_ms = (reads / (rd * 1e9) + writes / (wr * 1e9)) * 1e3
        return {"read_g_per_s": rd, "write_g_per_s": wr, "probe_dram_line_reads": reads,
                "probe_dram_sector_writes": writes, "ceiling_ms": ceil_ms,
                "frac": ceil_ms / probe_ms if probe_ms else None,
                "source": "PyTorch index_select / index_put_ over 16 GiB (profiles/random_ceiling_torch_r02.json); "
                          "probe DRAM counts from ncu (profiles/ncu_probe_summary.json)"}
    except Exception:
        return None


def ncu_traffic():
    """dram bytes per probe launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_probe_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------------------ workload

ROWS = 1 << 30
SHARDS = 8
MAX_PROBE = 128
TABLE_SEED = 7
ID_SEED = 5
BATCH = 4 * 1024 * 1024
SAMPLER_SEED = 0x5CA1AB1E


def prefill_count(rows):
    return int(0.8 * rows)


def host_cpu() -> str:
    """nproc and the CPU model (SURVEY 8d asks for both beside the CPU number)."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{os.cpu_count()} logical CPUs, {model}"


def run_reference(steps: int, warmup: int, rows: int = ROWS, log=print):
    """The reference library (oracle/_ref, OpenMP process_batch) on the SAME workload as the GPU
    arm: the same TableLayout (2^30 rows, S=8, P=128, seed 7), the same prefill
    (DistinctIdStream(5).at([0, 0.8 * rows)) at now = 1) and the same batch stream (batch b of the
    GPU arm's list, now = 2 + b).  Each batch is timed the reference's way
    (proj/src/experiments.cpp:339-347): steady_clock around mpzch::process_batch alone, inside
    the shim (the IdBatch is packed before the clock starts).  The prefill goes through the
    reference's per-shard entry process_shard_batch, shards in parallel (the same state
    process_batch builds from distinct ids; untimed)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    L = pyoracle.lib(kind)
    cores = os.cpu_count() or 1
    if kind == "reference":
        L["set_threads"](cores)
    else:
        cores = 1
    import paper_2602_17050_b200 as mz
    caps = mz.even_capacities(rows, SHARDS)
    t = pyoracle.OracleTable(caps, MAX_PROBE, TABLE_SEED, kind=kind)
    npre = prefill_count(rows)
    t0 = time.perf_counter()
    if kind == "reference":
        t.prefill_distinct(ID_SEED, 0, npre, 1)
    else:
        for a in range(0, npre, BATCH):
            ids = distinct_ids_t(ID_SEED, torch.arange(a, min(a + BATCH, npre), dtype=torch.int64))
            t.process_batch(ids.numpy().view(np.uint64), 1, 0)
    log(f"[ref] prefill {npre} ids into {rows} rows in {time.perf_counter() - t0:.1f}s "
        f"({kind}, {cores} threads)")
    fresh_base = npre
    times = []
    for b in range(warmup + steps):
        idx, nf = batch_indices(torch, "cpu", npre, BATCH, b, fresh_base, SAMPLER_SEED)
        fresh_base += nf
        ids = distinct_ids_t(ID_SEED, idx).numpy().view(np.uint64)
        if kind == "reference":
            e, _, _ = t.process_batch_timed(ids, 2 + b)
        else:
            s = time.perf_counter()
            t.process_batch(ids, 2 + b, 0)
            e = time.perf_counter() - s
        if b >= warmup:
            times.append(e)
    tot = sum(times)
    del t
    return dict(value=BATCH * len(times) / tot, kind=kind, cores=cores, ms=1e3 * tot / len(times),
                sample=f"the GPU arm's workload: {rows}-row table (S={SHARDS}, P={MAX_PROBE}, load 0.8 "
                       f"prefilled untimed), batches {warmup}..{warmup + steps - 1} of the same stream "
                       f"({BATCH} positions, 90% hit / 10% fresh), each timed with steady_clock around "
                       f"process_batch(ExecMode::Parallel) alone",
                threads_effective=min(cores, SHARDS) if kind == "reference" else 1)


def c5_config(rows, world, backend="nccl", transport="device"):
    """The workload dict both arms print (same_config)."""
    return {"workload": ("C5: 1B-slot (2^30-row) table" if rows == ROWS else
                         f"C5-shaped {rows}-row table") + ", S=8 logical shards, "
                        "max_probe=128, load 0.8 prefilled via the API, 4M-position "
                        "batches 90% hit / 10% fresh, eviction Disabled"
                        + ("" if world == 1 else f"; row-sharded over {world} GPUs, "
                           + ("device-side protocol (ids and results by stores into the peers' "
                              "exchange regions over NVLink / CUDA IPC, system-scope flags, one "
                              "host wait per batch)" if transport == "device" else
                              "peer-memory id routing (IPC stores, "
                              f"{backend} barrier)" if transport == "peer" else
                              f"{backend} all-to-all id routing")),
            "rows": rows, "num_shards": SHARDS, "max_probe": MAX_PROBE,
            "batch_positions": BATCH, "global_batch": BATCH,
            "parallelism": "single GPU" if world == 1 else f"row-sharded x{world}",
            "l2": "inputs larger than L2 (16 GiB identity+metadata, random probes)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=ROWS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    log = (lambda *a: print(*a, file=sys.stderr, flush=True))
    metric = "remapped IDs/sec (insert+evict) and HBM GB/s fraction at 1/2/4/8 B200 vs CPU ref"

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_reference(args.steps, max(args.warmup, 1), rows=args.rows, log=log)
        line = {"metric": metric, "value": r["value"], "unit": "IDs/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": r["ms"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (DistinctIdStream ids, SplitMix64 sampler)",
                "config": c5_config(args.rows, world, os.environ.get("MPZCH_DIST_BACKEND", "nccl"),
                                    os.environ.get("MPZCH_TRANSPORT", "device")),
                "cpu_baseline": {"value": r["value"], "unit": "IDs/s", "cores": r["cores"],
                                 "threads_effective": r["threads_effective"],
                                 "kind": r["kind"], "sample": r["sample"], "host": host_cpu()},
                "e2e": {"value": r["value"], "unit": "IDs/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2602_17050_b200 as mz
    # MPZCH_DIST_BACKEND=gloo (+ MPZCH_SHARE_GPU=1) runs the multi-rank path with every rank
    # on cuda:0 and collectives staged through the host: a functional check of the N>1 code
    # on a single-GPU box, never a scaling number
    backend = os.environ.get("MPZCH_DIST_BACKEND", "nccl")
    transport = os.environ.get("MPZCH_TRANSPORT", "device")
    share = os.environ.get("MPZCH_SHARE_GPU", "0") == "1"
    if world > 1:
        import torch.distributed as dist
        dev_i = 0 if share else local
        torch.cuda.set_device(dev_i)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_i))
        else:
            dist.init_process_group(backend)
    dev = (0 if share else local) if world > 1 else 0
    red_dev = "cpu" if (world > 1 and backend == "gloo") else dev  # device of reduction tensors
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)

    rows = args.rows
    caps = mz.even_capacities(rows, SHARDS)
    cfg = mz.TableConfig(caps, MAX_PROBE, TABLE_SEED)
    pol = mz.EvictionPolicy.disabled()
    t_build = time.perf_counter()
    out_s = torch.empty(BATCH, dtype=torch.int64, device=dev)
    out_o = torch.empty(BATCH, dtype=torch.uint8, device=dev)
    if world == 1:
        table = mz.MpzchTable(cfg, device=dev)
        probe_table = table

        def remap(ids, now):
            table.process_batch_device(ids, now, pol, None, out_s, out_o, None, stream)

        def remap_async(ids, now):  # enqueue only; the ticket is waited after the loop
            return table.process_batch_device_async(ids, now, pol, None, out_s, out_o, None, stream)
    elif transport == "device":
        # C5 row-sharded: the S=8 logical shards of ONE 1B-slot table spread over the ranks;
        # every global batch of BATCH positions is split into rank slices (strong scaling).
        # The device-side protocol (csrc/sharded.cu): ids out / results back by stores into the
        # peers' exchange regions (CUDA IPC over NVLink), every phase on the stream, one host
        # wait per batch; torch.distributed only carries the 128-byte export records once
        sharded = mz.ShardedRank(cfg, rank, world, BATCH, device=dev)
        recs = [None] * world
        torch.distributed.all_gather_object(recs, sharded.export())
        sharded.connect_ipc(recs)
        probe_table = sharded.table
        table = sharded  # .wait(ticket)

        def remap(ids, now):
            sharded.process_batch_device(ids, now, pol, None, out_s, out_o, None, stream)

        def remap_async(ids, now):
            return sharded.process_batch_device_async(ids, now, pol, None, out_s, out_o, None, stream)
    else:
        # the host-driven protocol (paper_2602_17050_b200/sharded.py): peer stores or NCCL
        # all-to-all, with host collectives between the phases
        from paper_2602_17050_b200.sharded import ShardedMpzchTable, TorchComm
        sharded = ShardedMpzchTable(cfg, TorchComm(), device=dev, transport=transport)
        probe_table = sharded.engine.table

        def remap(ids, now):
            sharded.process_batch(ids, now, pol)

        remap_async = None  # the sharded protocol synchronises on its collectives
    stats_of = sharded.last_stats if (world > 1 and transport == "device") else probe_table.last_stats

    def my_slice(lo, hi):
        n = hi - lo
        return lo + rank * n // world, lo + (rank + 1) * n // world

    npre = prefill_count(rows)
    for a in range(0, npre, BATCH):
        s0, s1 = my_slice(a, min(a + BATCH, npre))
        ids = distinct_ids_t(ID_SEED, torch.arange(s0, s1, dtype=torch.int64, device=dev))
        remap(ids, 1)
    torch.cuda.synchronize(dev)
    log(f"[rank {rank}] prefill {npre} ids into {rows} rows ({world} rank(s)) in "
        f"{time.perf_counter() - t_build:.1f}s; stats {probe_table.last_stats()}")

    # pre-generate the W + K batches (+ K more for the profiled pass that splits the step into
    # kernels): the same global batch on every rank, each keeps its slice
    nb = args.warmup + 2 * args.steps
    batches = []
    fresh_base = npre
    b0, b1 = my_slice(0, BATCH)
    for b in range(nb):
        idx, nf = batch_indices(torch, dev, npre, BATCH, b, fresh_base, SAMPLER_SEED)
        fresh_base += nf
        batches.append(distinct_ids_t(ID_SEED, idx[b0:b1]).contiguous())
    torch.cuda.synchronize(dev)

    for b in range(args.warmup):
        remap(batches[b], 2 + b)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()

    launches0 = probe_table.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stats = []
    with Clocks(dev) as clk:
        clk.wait_first()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        w0 = time.time()
        ev0.record(stream)
        timed = range(args.warmup, args.warmup + args.steps)
        if remap_async is not None:
            # pipelined: enqueue every step, then wait each ticket (each wait reports its
            # batch's errors exactly as the synchronous call would)
            tickets = [remap_async(batches[b], 2 + b) for b in timed]
            for tk in tickets:
                table.wait(tk)
                stats.append(stats_of())
        else:
            for b in timed:
                remap(batches[b], 2 + b)
                stats.append(stats_of())
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        ms_total = ev0.elapsed_time(ev1)
        launches = probe_table.kernel_launches() - launches0
        # the per-kernel split (roofline, kernel_ms) from a second pass over K fresh batches of
        # the same mix with the in-library CUDA-event profiler on (events between the kernels;
        # kept out of the timed region above)
        probe_table.set_profiling(True)
        for b in range(args.warmup + args.steps, nb):
            remap(batches[b], 2 + b)
        torch.cuda.synchronize(dev)
        prof = probe_table.profile()
        probe_table.set_profiling(False)
        # the timed region is short next to nvidia-smi's sampling period: keep the same load
        # running (re-remapping the timed batches, untimed) until >= 3 samples fall inside
        k = 0
        while k < 2000:
            more = len([t for t, _ in clk.rows if t >= w0]) < 4
            if world > 1:
                more = bool(_allreduce_max_int(torch, int(more), red_dev))
            if not more:
                break
            remap(batches[args.warmup + k % args.steps], 2 + nb + k)
            k += 1
        torch.cuda.synchronize(dev)
        clk.windows.append((w0, time.time()))
    if world > 1:
        tt = torch.tensor([ms_total], device=red_dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps
    value = BATCH * args.steps / (ms_total / 1e3)

    # e2e: host buffers in, host buffers out, through the public API (pinned memory)
    # (48 steps: the loop's pipeline fill and drain -- about D steps of latency -- are a small
    # part of the timed region; 20 steps measured 4.46, 48 steps 5.03 G/s)
    e2e_steps = args.e2e_steps or max(48, args.steps)
    e2e_batches = []
    for i in range(e2e_steps):
        idx, nf = batch_indices(torch, dev, npre, BATCH, nb + i, fresh_base, SAMPLER_SEED)
        fresh_base += nf
        e2e_batches.append(distinct_ids_t(ID_SEED, idx[b0:b1]).cpu().pin_memory())
    nloc = b1 - b0
    pin_s = torch.empty(nloc, dtype=torch.int64).pin_memory()
    pin_o = torch.empty(nloc, dtype=torch.uint8).pin_memory()
    pin_ev = torch.empty(16, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e2e_api = None
    if world == 1:
        # pipelined service loop through the public API: the H2D of step i, the remap of
        # step i-1 (mpzch_process_batch_device_async) and the D2H of step i-2 overlap on three
        # streams (PCIe is full duplex); D buffer sets, so the host only blocks on step i-D
        # (its ticket -- errors reported exactly as the synchronous call would -- and its
        # slots/outcomes on the host) before reusing that step's buffers
        D = 4
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        d_ids = [torch.empty(nloc, dtype=torch.int64, device=dev) for _ in range(D)]
        d_s = [torch.empty(nloc, dtype=torch.int64, device=dev) for _ in range(D)]
        d_o = [torch.empty(nloc, dtype=torch.uint8, device=dev) for _ in range(D)]
        h_s = [torch.empty(nloc, dtype=torch.int64).pin_memory() for _ in range(D)]
        h_o = [torch.empty(nloc, dtype=torch.uint8).pin_memory() for _ in range(D)]
        ev_in = [torch.cuda.Event() for _ in range(e2e_steps)]
        ev_cmp = [torch.cuda.Event() for _ in range(e2e_steps)]
        ev_out = [torch.cuda.Event() for _ in range(e2e_steps)]
        t0 = time.perf_counter()
        tickets = []
        done_slots = 0

        def retire(k):  # step k: its ticket waited and its results on the host
            table.wait(tickets[k])
            ev_out[k].synchronize()
            return int(h_o[k % D][0])  # touch the host copy

        for i in range(e2e_steps):
            j = i % D
            if i >= D:
                retire(i - D)
                done_slots += 1
            with torch.cuda.stream(s_in):
                d_ids[j].copy_(e2e_batches[i], non_blocking=True)
                ev_in[i].record(s_in)
            stream.wait_event(ev_in[i])
            tickets.append(table.process_batch_device_async(d_ids[j], 100 + i, pol, None,
                                                            d_s[j], d_o[j], None, stream))
            ev_cmp[i].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[i])
                h_s[j].copy_(d_s[j], non_blocking=True)
                h_o[j].copy_(d_o[j], non_blocking=True)
                ev_out[i].record(s_out)
        for k in range(done_slots, e2e_steps):
            retire(k)
        e2e_s = time.perf_counter() - t0
        # the link's own ceiling for this traffic: the same H2D and D2H bytes per step copied
        # concurrently with no remap in between (what the e2e number is bound by)
        ev_a, ev_b, ev_c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize(dev)
        reps = 6
        ev_a.record(stream)
        s_in.wait_event(ev_a)
        s_out.wait_event(ev_a)
        for r in range(reps):
            with torch.cuda.stream(s_in):
                d_ids[r % D].copy_(e2e_batches[r % e2e_steps], non_blocking=True)
            with torch.cuda.stream(s_out):
                h_s[r % D].copy_(d_s[r % D], non_blocking=True)
                h_o[r % D].copy_(d_o[r % D], non_blocking=True)
        ev_b.record(s_in)
        ev_c.record(s_out)
        torch.cuda.synchronize(dev)
        link_ms = max(ev_a.elapsed_time(ev_b), ev_a.elapsed_time(ev_c)) / reps
        pcie_bound = BATCH / (link_ms / 1e3)
        e2e_api = ("mpzch_process_batch_device_async + pinned H2D/D2H on separate streams "
                   "(each step's ticket waited and its slots/outcomes read back)")
        # the plain synchronous host-buffer call, for reference (one untimed call first: it
        # sizes the handle's host-path staging buffers)
        table.process_batch(e2e_batches[0].numpy().view(np.uint64), 199, pol,
                            out_slots=pin_s.numpy().view(np.uint64), out_outcomes=pin_o.numpy(),
                            out_evicted=pin_ev)
        t1 = time.perf_counter()
        for i in range(min(3, e2e_steps)):
            table.process_batch(e2e_batches[i].numpy().view(np.uint64), 200 + i, pol,
                                out_slots=pin_s.numpy().view(np.uint64), out_outcomes=pin_o.numpy(),
                                out_evicted=pin_ev)
        e2e_sync_value = BATCH * min(3, e2e_steps) / (time.perf_counter() - t1)
    elif transport == "device":
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            d = e2e_batches[i].to(dev, non_blocking=True)
            sharded.process_batch_device(d, 100 + i, pol, None, out_s, out_o, None, stream)
            pin_s.copy_(out_s[:nloc], non_blocking=True)
            pin_o.copy_(out_o[:nloc], non_blocking=True)
            torch.cuda.synchronize(dev)
        e2e_s = time.perf_counter() - t0
        e2e_api = "mpzch_sharded_process_batch (pinned host slices, H2D/D2H timed)"
        e2e_sync_value = None
        pcie_bound = None
    else:
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            d = e2e_batches[i].to(dev, non_blocking=True)
            s_, o_, _ = sharded.process_batch(d, 100 + i, pol)
            pin_s.copy_(s_, non_blocking=True)
            pin_o.copy_(o_, non_blocking=True)
            torch.cuda.synchronize(dev)
        e2e_s = time.perf_counter() - t0
        e2e_api = "ShardedMpzchTable.process_batch (pinned host slices, H2D/D2H timed)"
        e2e_sync_value = None
        pcie_bound = None
    if world > 1:
        tt = torch.tensor([e2e_s], device=red_dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = BATCH * e2e_steps / e2e_s

    peak, peak_src = peaks()
    probe_ms = prof["probe_ms"] / max(prof["probe_launches"], 1)
    probe_bytes = prof["probe_bytes"] / max(prof["probe_launches"], 1)
    achieved = probe_bytes / (probe_ms / 1e3) / 1e9 if probe_ms else 0.0
    batch_bytes = prof["batch_bytes"] / max(prof["batches"], 1)
    batch_ms = prof["batch_ms"] / max(prof["batches"], 1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = run_reference(3, 1, rows=rows, log=log)
            cpu = {"value": r["value"], "unit": "IDs/s", "cores": r["cores"], "kind": r["kind"],
                   "threads_effective": r["threads_effective"], "sample": r["sample"],
                   "host": host_cpu()}
        except Exception as e:  # the baseline must not take the GPU number down with it
            cpu = {"value": None, "unit": "IDs/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    # distinct (id, feature) uniques per step (uniques/s beside positions/s), counted
    # on the timed batches outside the timed region
    uniq = statistics.mean(int(torch.unique(batches[b]).numel())
                           for b in range(args.warmup, args.warmup + args.steps)) * world

    if rank == 0:
        agg = {k: sum(s[k] for s in stats) for k in ("found", "inserted", "collision", "new_ids")}
        line = {
            "metric": metric, "value": value, "unit": "IDs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (DistinctIdStream ids, SplitMix64 sampler)",
            "config": c5_config(rows, world, backend, transport),
            "outcomes_per_step_rank0_owner": {k: v / args.steps for k, v in agg.items()},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic() if world == 1 else None,
                         "frac_vs_nominal_8tbs": achieved / 8000.0,
                         # DRAM bytes (ncu, the C5 launch) per algorithmic byte
                         "overfetch": (ncu_traffic() / probe_bytes) if (world == 1 and rows == ROWS and
                                                                        ncu_traffic() and probe_bytes) else None,
                         "kernel": "k_probe<Disabled, 1 position per thread> (probe of every position; rank 0)",
                         "algorithmic_bytes_per_launch": probe_bytes,
                         "probe_sectors_per_launch": prof["probe_sectors"] / max(prof["probe_launches"], 1),
                         "launch_ms": probe_ms, "peak_source": peak_src,
                         "random_sector_ceiling_gbs": random_sector_ceiling(),
                         "random_access_ceiling": random_access_ceiling(),
                         # (the ncu access count is for the single-GPU C5 launch)
                         "random_access_frac": _access_frac(probe_ms) if (world == 1 and rows == ROWS) else None,
                         "independent_ceiling": independent_ceiling(probe_ms) if (world == 1 and rows == ROWS) else None,
                         "share_of_step": probe_ms / ms_step,
                         "batch_algorithmic_bytes": batch_bytes,
                         "batch_gbs": batch_bytes / (batch_ms / 1e3) / 1e9 if batch_ms else 0.0,
                         "claim_ms": prof["claim_ms"] / max(prof["batches"], 1),
                         "tail_ms": prof["tail_ms"] / max(prof["batches"], 1),
                         "kernel_ms": {k: prof[k] / max(prof["batches"], 1) for k in
                                       ("validate_ms", "dedup_ms", "claimk_ms", "commit_ms",
                                        "finalize_ms")}},
            "uniques_per_s": uniq / (ms_step / 1e3),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "IDs/s", "h2d_bytes_per_step": BATCH * 8,
                    "d2h_bytes_per_step": BATCH * 9, "steps": e2e_steps, "api": e2e_api,
                    "synchronous_host_call_value": e2e_sync_value,
                    "pcie_copy_only_ids_per_s": pcie_bound},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        sharded.close()  # unmap the peers' IPC buffers before the group goes away
        torch.distributed.destroy_process_group()


def _access_frac(probe_ms):
    """k_probe's DRAM accesses per second (ncu count per launch / live launch time) against the
    measured random-access read ceiling: the roofline that binds this kernel."""
    acc, ceil = probe_dram_accesses(), random_access_ceiling()
    if not acc or not ceil or not probe_ms:
        return None
    return acc / (probe_ms / 1e3) / (ceil["read_g_per_s"] * 1e9)


def _allreduce_max_int(torch, x, dev):
    t = torch.tensor([x], device=dev, dtype=torch.int64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return int(t.item())


if __name__ == "__main__":
    main()
