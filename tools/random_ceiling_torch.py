"""Independent check of the random-access ceiling with library kernels (PyTorch's own
index_select / index_put_, nothing of this repo): uniform random 8 B / 32 B / 128 B gathers and
random 8 B / 32 B scatters over arrays of 1-16 GiB on one B200, CUDA-event timed, reported as
G accesses/s next to the ceiling tools/sector_probe.cu measured (~36 G/s at 16 GiB).

    python tools/random_ceiling_torch.py [--out gpurun_out/random_ceiling_torch.json]
"""
import argparse
import json

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = []
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        b.synchronize()
        best.append(a.elapsed_time(b))
    best.sort()
    return best[len(best) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/random_ceiling_torch.json")
    ap.add_argument("--n", type=int, default=1 << 24, help="accesses per launch")
    args = ap.parse_args()
    dev = torch.device("cuda")
    rows = []
    for gib in (1, 4, 16):
        words = gib << 27  # int64 words
        a = torch.empty(words, dtype=torch.int64, device=dev)
        a.fill_(1)
        for width in (8, 32, 128):
            per = width // 8
            view = a.view(-1, per)
            idx = torch.randint(0, view.shape[0], (args.n,), device=dev)
            ms = timed(lambda: torch.index_select(view, 0, idx))
            rows.append({"gib": gib, "op": f"index_select {width} B rows", "accesses": args.n, "ms": ms,
                         "G_accesses_s": args.n / ms / 1e6, "useful_gbs": args.n * width / ms / 1e6})
        for width in (8, 32):
            per = width // 8
            view = a.view(-1, per)
            idx = torch.randint(0, view.shape[0], (args.n,), device=dev)
            src = torch.ones(args.n, per, dtype=torch.int64, device=dev)
            ms = timed(lambda: view.index_put_((idx,), src))
            rows.append({"gib": gib, "op": f"index_put_ {width} B rows", "accesses": args.n, "ms": ms,
                         "G_accesses_s": args.n / ms / 1e6, "useful_gbs": args.n * width / ms / 1e6})
        del a
        torch.cuda.empty_cache()
    for r in rows:
        print(f"{r['gib']:>3} GiB  {r['op']:<26} {r['ms']:8.3f} ms  {r['G_accesses_s']:6.2f} G/s  "
              f"{r['useful_gbs']:8.1f} GB/s")
    with open(args.out, "w") as f:
        json.dump({"what": "random gathers/scatters with PyTorch's own kernels (independent of this repo's code)",
                   "device": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
