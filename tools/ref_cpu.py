"""The unmodified reference (`dgmg` from baseline/_ref) on the BASELINE
configs, all host threads and one thread: one JSON line per (config,
threads) with the per-step time of `LevelSmoother.smooth` (setup excluded).

    python tools/ref_cpu.py [--configs 1,2,4] [--reps 3] [--one-thread 1,2,4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from threadpoolctl import threadpool_limits  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4,5")
ap.add_argument("--one-thread", default="1,2,4", help="configs also timed with one BLAS thread")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cores = len(os.sched_getaffinity(0))
one = {int(c) for c in a.one_thread.split(",") if c}
for c in (int(v) for v in a.configs.split(",")):
    cfg = bench.CONFIGS[c]
    step = bench.RefStep(cfg, (cfg["nc"],) * cfg["d"])
    for threads in ([cores, 1] if c in one else [cores]):
        with threadpool_limits(limits=threads):
            step()  # warm-up
            reps = a.reps if c in (1, 2, 4) else 1
            times = [step() for _ in range(reps)]
        t = min(times)
        print(json.dumps({"config": c, "workload": cfg["name"], "threads": threads,
                          "cpu_model": bench._cpu_model(), "ndofs": step.ndofs,
                          "setup_s": step.setup_s, "step_s": t, "dof_per_s": step.ndofs / t,
                          "reps": reps}), flush=True)
