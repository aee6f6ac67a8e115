"""Host<->device copy bandwidth from pinned memory, one direction at a time
and both directions at once (the e2e step's bound).

    python tools/pcie_duplex.py
"""
import json

import torch


def run():
    n = 453_000_000 // 8  # one cfg-5 vector
    h_in = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(h2d, d2h, reps=5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            s_in.wait_event(e0) if False else None
            with torch.cuda.stream(s_in):
                for k in range(h2d):
                    d[k].copy_(h_in[k], non_blocking=True)
            with torch.cuda.stream(s_out):
                for _ in range(d2h):
                    h_out.copy_(d[2], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s_in)
        torch.cuda.current_stream().wait_stream(s_out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gb = (h2d + d2h) * n * 8 / 1e9
        return {"h2d_vectors": h2d, "d2h_vectors": d2h, "ms": ms, "gbs_total": gb / ms * 1e3}

    timed(1, 1, 1)
    for h2d, d2h in ((2, 0), (0, 1), (2, 1), (2, 2)):
        print(json.dumps(timed(h2d, d2h)), flush=True)


if __name__ == "__main__":
    run()
