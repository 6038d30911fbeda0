"""e2e (as_spmv_host) sweep on C2 (developer tool): PCIe copy references (H2D alone, D2H alone,
both on two streams) and the pipelined host SpMV for ROW_DIV(k bands) { DIA } over k."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2212_10432_b200 as asp  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    c = synth.c2_lap2d(2048)
    A = asp.Matrix.from_coo(c.m, c.n, c.row, c.col, c.val)
    x, _ = synth.vectors(c.n, c.m, 2)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.zeros(c.m, dtype=torch.float64).pin_memory()
    xd = torch.empty(c.n, dtype=torch.float64, device="cuda")
    yd = torch.empty(c.m, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {"h2d_ms": timed(lambda: xd.copy_(xh, non_blocking=True)),
           "d2h_ms": timed(lambda: yh.copy_(yd, non_blocking=True))}

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s2):
            yh.copy_(yd, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    out["both_ms"] = timed(both)
    xn, yn = xh.numpy(), yh.numpy()
    dia = "DIA_DECOM(theta=0.5,max=8) { DIA; SET_RESOURCE(tpb=128,grid=16,stages=0) }"
    for k in (1, 2, 4, 8, 16, 32, 64):
        g = dia if k == 1 else "ROW_DIV(cuts=[%s]) { %s }" % (",".join(str(c.m * i // k) for i in range(1, k)), dia)
        P = asp.Plan(A, g, device=0)
        out[f"bands{k}_ms"] = timed(lambda: P.spmv_host(1.0, xn, 0.0, yn))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
