#!/usr/bin/env python
"""Host<->device copy rates on this box (pinned host memory, cudaMemcpyAsync
through torch copy_): H2D alone, D2H alone, and both at once on two streams —
the ceiling of bench.py's e2e leg, which moves ~805 MB up and ~671 MB down per
C2 step.

    python tools/pcie_probe.py [--mb 256] [--reps 8]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=256)
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    n = args.mb * 2**20
    h_up = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dn = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}

    def run(up, down):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        for _ in range(args.reps):
            if up:
                with torch.cuda.stream(s1):
                    d_up.copy_(h_up, non_blocking=True)
            if down:
                with torch.cuda.stream(s2):
                    h_dn.copy_(d_dn, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    run(True, True)
    for name, up, down in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
        t = run(up, down)
        res[name + "_GBps"] = n * args.reps / t / 1e9
    res["note"] = "both: per-direction rate with H2D and D2H concurrent"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
