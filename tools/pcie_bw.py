"""Host<->device copy bandwidth with pinned buffers (developer measurement for the e2e
number): H2D alone, D2H alone, and both directions at once on two streams.

    python tools/pcie_bw.py [--mb 64] > gpurun_out/pcie.json
"""
import argparse
import json
import statistics


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=64)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    n = args.mb << 20
    h_up = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dn = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        ts = []
        for _ in range(args.reps + 3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts[3:])

    def up():
        d_up.copy_(h_up, non_blocking=True)

    def down():
        h_dn.copy_(d_dn, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_up.copy_(h_up, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dn.copy_(d_dn, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_up, t_dn, t_both = timed(up), timed(down), timed(both)
    gb = n / 1e9
    print(json.dumps({"mb": args.mb, "h2d_ms": t_up, "d2h_ms": t_dn, "both_ms": t_both,
                      "h2d_gbs": gb / (t_up * 1e-3), "d2h_gbs": gb / (t_dn * 1e-3),
                      "both_gbs_total": 2 * gb / (t_both * 1e-3)}))


if __name__ == "__main__":
    main()
