"""Benchmark: fp64 Schwarz smoothing DoFs/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Workload (default, BASELINE.json configs[4], the config quoted at 1/2/4/8
GPUs): 3D Q5 SIPG Laplacian, additive vertex-patch Schwarz (12^3-DoF patches,
16 structured colours, omega = 0.25) plus the matrix-free residual, fp64,
64^3 cells per GPU; at N GPUs the box is 64 x 64 x 64N cells split in slabs
along z with two ghost layers exchanged by NCCL (weak scaling).  A step is one
additive smoothing step x <- x + omega sum_j R_j^T A_j^-1 R_j (b - A x).
`--config 1..4` selects the other BASELINE configs (1 GPU only).

Inputs: b, x0 ~ U[-1,1] from seeds 0/1 (synthetic); every vector
(453 MB at cfg 5) is larger than the 126 MB L2, so no L2 flush is needed.

`value` is device-timed (CUDA events, max over ranks) with inputs resident in
HBM; `e2e` times the public API (`LevelSmoother.smooth`) with the host->device
copy of x and b from pinned memory and the device->host copy of x inside the
timed region.  `--impl reference` times the reference itself (the unmodified
`dgmg` package, pip-installed by `build()` into the git-ignored `baseline/_ref`,
which travels to the GPU box) on the host cores, `LevelSmoother.smooth` on the
same level; `cpu_baseline` in our line is the same measurement (one step).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(d=2, nc=64, k=3, kind="acs", omega=0.7,
            name="cfg1: 2D Q3 SIPG, 64^2 cells, additive cell Schwarz (ACS)"),
    2: dict(d=3, nc=32, k=3, kind="avs", omega=0.25,
            name="cfg2: 3D Q3 SIPG, 32^3 cells, additive vertex-patch Schwarz (AVS, 16 colours)"),
    3: dict(d=3, nc=32, k=7, kind="mvs", omega=1.0,
            name="cfg3: 3D Q7 SIPG, 32^3 cells, multiplicative vertex-patch sweep (MVS, 16 colours)"),
    4: dict(d=3, nc=16, k=15, kind="acs", omega=0.7,
            name="cfg4: 3D Q15 SIPG, 16^3 cells, additive cell Schwarz (ACS)"),
    5: dict(d=3, nc=64, k=5, kind="avs", omega=0.25,
            name="cfg5: 3D Q5 SIPG, 64^3 cells per GPU (64x64x64N slabs), AVS 12^3-DoF patches, 16 colours"),
}
METRIC = "fp64 Schwarz smoothing DoFs/s (1/2/4/8 B200) + % fp64/HBM roofline"
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def _fp64_peak():
    """Measured fp64 peak (DMMA.8x8x4 loop, tools/microbench/fp64_peak.cu)."""
    best = None
    try:
        with open(FP64_PEAK_FILE) as f:
            for line in f:
                rec = json.loads(line)
                if "tflops" in rec:
                    best = max(best or 0.0, rec["tflops"])
    except (OSError, ValueError):
        pass
    return (best, "measured fp64 DMMA burst, profiles/r01_fp64_peak.json") if best else \
        (37.0, "nominal fp64 (no measurement file)")


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def _load_reference():
    """The unmodified reference package `dgmg`, installed by `build()` into the
    git-ignored `baseline/_ref` (pip --target of /root/reference/pkg; it
    travels to the GPU box with the snapshot).  None when absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "dgmg")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import dgmg  # noqa: F401
    from dgmg import dgop, mesh, polybasis, smoothers
    if not os.path.abspath(dgop.__file__).startswith(os.path.abspath(REF_DIR)):
        raise RuntimeError(f"dgmg imported from {dgop.__file__}, not {REF_DIR}")
    return mesh, polybasis, dgop, smoothers


class RefStep:
    """One smoothing step of the reference itself on `dims` cells:
    `mesh.build_hierarchy(d, n_c, 0)`, `make_context`, `make_level_smoother(ctx, basis, SmootherConfig(kind,
    omega))`, then `LevelSmoother.smooth(x, b)` on the seeded inputs
    (reference `smoothers.py:131-197`, `dgop.py:399-411`)."""

    def __init__(self, cfg, dims):
        mods = _load_reference()
        if mods is None:
            raise FileNotFoundError("baseline/_ref/dgmg not installed")
        mesh, polybasis, dgop, smoothers = mods
        d, k = cfg["d"], cfg["k"]
        t0 = time.perf_counter()
        if len(set(dims)) != 1:
            raise ValueError("the reference builds cubes only (mesh.py:142-157)")
        lvl = mesh.build_hierarchy(d, dims[0], 0).levels[0]
        basis = polybasis.Basis1D.make(k)
        self.ctx = dgop.make_context(lvl, basis, 1.0)
        self.sm = smoothers.make_level_smoother(
            self.ctx, basis, smoothers.SmootherConfig(kind=cfg["kind"], omega=cfg["omega"]))
        self.setup_s = time.perf_counter() - t0
        self.ndofs = self.ctx.ndofs
        self.b = np.random.default_rng(0).uniform(-1.0, 1.0, self.ndofs)
        self.x0 = np.random.default_rng(1).uniform(-1.0, 1.0, self.ndofs)

    def __call__(self):
        x = self.x0.copy()
        t0 = time.perf_counter()
        self.sm.smooth(x, self.b)
        return time.perf_counter() - t0


class PortStep:
    """Fallback when baseline/_ref is missing: the oracle port (numpy)."""

    def __init__(self, cfg, dims):
        from oracle.sipg_oracle import OracleLevel, seeded_inputs
        t0 = time.perf_counter()
        self.lvl = OracleLevel(tuple(dims), cfg["k"], h=1.0 / dims[0])
        self.setup_s = time.perf_counter() - t0
        self.ndofs = self.lvl.ndofs
        self.x0, self.b = seeded_inputs(self.ndofs, 0)
        self.kind, self.omega = cfg["kind"], cfg["omega"]

    def __call__(self):
        t0 = time.perf_counter()
        self.lvl.smooth(self.kind, self.omega, self.x0, self.b)
        return time.perf_counter() - t0


def _cpu_step(cfg, dims):
    try:
        return RefStep(cfg, dims), "reference"
    except (FileNotFoundError, ImportError):
        return PortStep(cfg, dims), "port"


def config_dict(cfg, dims, ws, n_global, slab):
    """The `config` object both arms print (identical, so the driver's
    same-config check can hold)."""
    n_local = n_global // ws
    return {"workload": cfg["name"], "dims": list(dims), "k": cfg["k"], "kind": cfg["kind"],
            "omega": cfg["omega"], "global_dofs": n_global,
            "parallelism": f"slab{ws}" if slab else "single",
            "l2": "inputs larger than L2 (no flush)" if n_local * 8 > 126e6
            else "inputs smaller than L2"}


def _bench_dims(cfg, ws, slab):
    d, nc = cfg["d"], cfg["nc"]
    return (nc,) * d if not slab else (nc, nc, nc * ws)


def run_reference(args, cfg):
    """The reference's own CPU implementation (`dgmg`, unmodified, from
    baseline/_ref) timed on the box's host cores: W untimed + K timed
    `LevelSmoother.smooth` steps on the same level as our arm (rank 0 only;
    at N > 1 the per-GPU 64^3 share, since the CPU rate is size-independent
    and the 64x64x64N box does not fit a CPU process at N = 8)."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    slab = ws > 1 or args.slab
    dims = _bench_dims(cfg, ws, slab)
    run_dims = dims if not slab else (cfg["nc"],) * 3
    step, kind = _cpu_step(cfg, run_dims)
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    t = float(np.mean(times))
    value = step.ndofs / t
    cores = len(os.sched_getaffinity(0))
    what = "dgmg (unmodified reference, baseline/_ref)" if kind == "reference" else \
        "oracle port (baseline/_ref missing)"
    sample = (f"{what}: LevelSmoother.smooth on {'x'.join(map(str, run_dims))} cells "
              f"({step.ndofs} DoFs), one step per timed step; setup {step.setup_s:.1f} s excluded")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DoF/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1] b, x0)",
        "config": config_dict(cfg, dims, ws, step.ndofs * (ws if slab else 1), slab),
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": cores, "kind": kind,
                         "sample": sample, "cpu_model": _cpu_model(),
                         "blas_threads": cores, "min_ms": min(times) * 1e3,
                         "max_ms": max(times) * 1e3},
        "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(cfg, dims, budget_s=30.0):
    """The reference's step on the same level (rank 0, N = 1), all host
    threads: one step for the large configs (~20 s), up to 5 for small ones."""
    step, kind = _cpu_step(cfg, dims)
    times = []
    t_all = time.perf_counter()
    while True:
        times.append(step())
        if time.perf_counter() - t_all > budget_s or len(times) >= 5:
            break
    t = float(min(times))
    what = "dgmg (unmodified reference)" if kind == "reference" else "oracle port"
    return {"value": step.ndofs / t, "unit": "DoF/s", "cores": len(os.sched_getaffinity(0)),
            "kind": kind, "cpu_model": _cpu_model(),
            "sample": f"{what}: LevelSmoother.smooth on the full {'x'.join(map(str, dims))}-cell "
                      f"level, best of {len(times)} (setup {step.setup_s:.1f} s excluded)"}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1910_11239_b200 as dg
    from paper_1910_11239_b200 import flops as F

    ws, rank, local = _dist_env()
    if args.gpus != ws and ws > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    torch.cuda.set_device(local)
    slab = ws > 1 or args.slab
    if slab:
        # keep stdout to the one JSON line (NCCL prints its version otherwise)
        # (the image's Python starts with NCCL_DEBUG=VERSION, which prints the
        # version line on stdout: lower it, and send any NCCL log to stderr)
        # NCCL's init lines (ranks, nranks, transports) go to stderr for the
        # driver's log; an explicit NCCL_DEBUG setting is kept as given
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if not dist.is_initialized():
            if ws == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29531")
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            # a dead peer fails the run after 5 minutes instead of NCCL's 10-minute
            # default hanging the box (the halo exchange is the only traffic)
            import datetime
            dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                    timeout=datetime.timedelta(minutes=5))
    d, nc, k, kind, omega = cfg["d"], cfg["nc"], cfg["k"], cfg["kind"], cfg["omega"]
    if slab and args.config != 5:
        raise SystemExit("multi-GPU (slab) runs use the cfg-5 weak-scaling workload")
    dims = _bench_dims(cfg, ws, slab)

    if not slab:
        lvl = dg.build_hierarchy(d, nc, 0).levels[0]
        basis = dg.Basis1D.make(k)
        ctx = dg.make_context(lvl, basis, 1.0)
        sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=kind, omega=omega))
        n_local = ctx.ndofs
        step_obj = sm
    else:
        from paper_1910_11239_b200.distributed import SlabSmoother
        step_obj = SlabSmoother(dims, k, kind=kind, omega=omega, rank=rank, world=ws)
        n_local = step_obj.n_owned
    n_global = n_local * ws

    # seeded inputs generated on the host: seeds 0 / 1 on one GPU (the tests'
    # and the oracle's inputs); per-rank streams [0, rank] / [1, rank] on N > 1
    # (each rank only materialises its own slab)
    s_b, s_x = (0, 1) if ws == 1 else ([0, rank], [1, rank])
    b_h = np.random.default_rng(s_b).uniform(-1.0, 1.0, n_local)
    x_h = np.random.default_rng(s_x).uniform(-1.0, 1.0, n_local)
    stream = torch.cuda.current_stream()

    if not slab:
        x = torch.from_numpy(x_h).cuda()
        b = torch.from_numpy(b_h).cuda()

        def step():
            sm.smooth(x, b)
    else:
        step_obj.load(x_h, b_h)

        def step():
            step_obj.step()

    def barrier():
        if slab:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = int(step_obj.launches_per_step())
    clocks = ClockSampler(local)
    time.sleep(0.2)
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    if slab:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n_global / (ms_step * 1e-3)

    # ---- per-kernel split (dominant kernel for the roofline), direct launches
    kt = step_obj.kernel_times(reps=max(3, min(args.steps, 10)))
    rdims = dims if not slab else (nc, nc, nc)  # per-GPU share of the work
    flops_step, bytes_step = F.step_work(kind, d, k, rdims)
    if kind in ("avs", "mvs"):
        npatch = int(np.prod([v - 1 for v in rdims]))
        f_solve = F.solve_flops(d, 2 * (k + 1), npatch)
        dom = f"fdm2_kernel<{d},{2 * (k + 1)},patch> (patch solves: one launch, bulk reduce-add)"
    else:
        f_solve = F.solve_flops(d, k + 1, int(np.prod(dims)))
        dom = f"fdm2_kernel<{d},{k + 1},cell>"
    f_res = flops_step - f_solve
    peak, peak_src = _fp64_peak()
    hbm, hbm_src = _hbm_peak()
    if "flow_ms" in kt:
        # the whole step is one persistent dataflow kernel (residual + colours)
        dom = f"flow_kernel<{d},{k + 1}> (residual + all patch colours, one launch)"
        dom_ms, dom_f = kt["flow_ms"], flops_step
    else:
        solve_ms, res_ms = kt["solve_ms"], kt["residual_ms"]
        dom_ms, dom_f = (solve_ms, f_solve) if solve_ms >= res_ms else (res_ms, f_res)
        if solve_ms < res_ms:
            n1 = k + 1  # launch_res.cu: res3 for 3D n = 7..9 and n >= 13 by default
            res3 = d == 3 and os.environ.get("DGB_RES3", "1") != "0" and 7 <= n1 and (n1 <= 9 or n1 >= 13)
            dom = f"res3_kernel<{n1}> (residual)" if res3 else f"res2_kernel<{d},{n1}> (residual)"
    achieved = dom_f / (dom_ms * 1e-3) / 1e12
    # the kernels split interior-digit contractions even/odd (half the FMAs):
    # also report the fraction against the flops actually executed
    dev = step_obj.ctx.dev if not slab else step_obj._dev
    eo = getattr(dev, "eo", {"cell": False, "patch": False, "residual": False})
    eo_fdm = eo["cell"] if kind in ("acs", "mcs") else eo["patch"]
    fx_step = F.executed_step_flops(kind, d, k, rdims, eo_fdm, eo["residual"])
    dom_fx = dom_f * fx_step / flops_step
    traffic = None
    try:
        with open(TRAFFIC_FILE) as f:
            traffic = json.load(f).get(f"cfg{args.config}")
    except (OSError, ValueError):
        traffic = None
    # per-kernel fp64-pipe / issue / L1 utilisation of this config's step
    # kernels from the committed ncu capture (profiles/ncu_pipes.json)
    ncu_pipes = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_pipes.json")) as f:
            ncu_pipes = json.load(f).get(f"cfg{args.config}")
    except (OSError, ValueError):
        ncu_pipes = None

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not slab:
        # host vectors straight into the public API: LevelSmoother.smooth
        # copies x, b in and x out, pipelined in z-chunks against the kernels
        # (smoothers.LevelSmoother._host_step)
        xh = torch.from_numpy(x_h.copy()).pin_memory()
        bh = torch.from_numpy(b_h.copy()).pin_memory()
        for _ in range(2):
            sm.smooth(xh, bh)
        torch.cuda.synchronize()
        ke = max(3, min(args.steps, 20))
        e0.record(stream)
        for _ in range(ke):
            sm.smooth(xh, bh)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / ke
        e2e = {"value": n_global / (e_ms * 1e-3), "unit": "DoF/s",
               "h2d_bytes_per_step": 16 * n_local, "d2h_bytes_per_step": 8 * n_local,
               "ms_per_step": e_ms,
               "api": "LevelSmoother.smooth(pinned host tensors): H2D x,b / D2H x inside the call",
               "pipelined": bool(sm._pipelinable(xh, bh))}
        # the step's PCIe bound: the same copies alone (x, b in on one stream,
        # x out on another, concurrently), no kernels
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        xd = torch.empty(n_local, dtype=torch.float64, device="cuda")
        bd = torch.empty_like(xd)

        def copies():
            s_in.wait_stream(stream)
            s_out.wait_stream(stream)
            with torch.cuda.stream(s_in):
                xd.copy_(xh, non_blocking=True)
                bd.copy_(bh, non_blocking=True)
            with torch.cuda.stream(s_out):
                xh.copy_(sm._r, non_blocking=True)
            stream.wait_stream(s_in)
            stream.wait_stream(s_out)
        xsave = xh.clone()
        copies()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            copies()
        e1.record(stream)
        torch.cuda.synchronize()
        xh.copy_(xsave)
        c_ms = e0.elapsed_time(e1) / 3
        del xd, bd, xsave
        e2e["copy_bound_ms"] = c_ms
        e2e["frac_of_copy_bound"] = c_ms / e_ms
        # the reference's own callers pass pageable numpy arrays: the same
        # call on those (the copies go through the driver's staging buffers)
        # (first call: pageable copies; second call: the recurring buffers are
        # page-locked in place, _device.maybe_pin, its cost is in that call;
        # after that the call runs the pinned pipeline)
        xn, bn = x_h.copy(), b_h.copy()
        calls = []
        for _ in range(2):
            t0 = time.perf_counter()
            sm.smooth(xn, bn)
            calls.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize()
        kp = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(kp):
            sm.smooth(xn, bn)
        p_ms = (time.perf_counter() - t0) * 1e3 / kp
        from paper_1910_11239_b200 import _device
        e2e["pageable"] = {"value": n_global / (p_ms * 1e-3), "unit": "DoF/s", "ms_per_step": p_ms,
                           "first_call_ms": calls[0], "second_call_ms": calls[1],
                           "page_locked_in_place": bool(_device._pin_live),
                           "api": "LevelSmoother.smooth(numpy float64 arrays), the same arrays "
                                  "on every call as the reference's V-cycle passes them",
                           "timing": "host wall clock around the call (it returns with x final); "
                                     "first_call = pageable copies, second_call includes the "
                                     "in-place cudaHostRegister of x and b, ms_per_step = the "
                                     "calls after that"}
        del xn, bn
    else:
        e2e = step_obj.e2e(x_h, b_h, reps=max(3, min(args.steps, 10)))
        e2e["value"] = e2e.pop("dofs_local") * ws / (e2e["ms_per_step"] * 1e-3)
        t = torch.tensor([e2e["ms_per_step"]], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e["ms_per_step"] = float(t.item())
        e2e["value"] = n_global / (e2e["ms_per_step"] * 1e-3)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample(cfg, dims)

    if rank == 0:
        step_roof_ms = max(flops_step / (peak * 1e12), bytes_step / (hbm * 1e9)) * 1e3
        line = {
            "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform[-1,1] b, x0)",
            "config": config_dict(cfg, dims, ws, n_global, slab),
            "roofline": {"bound": "tensor", "pipe": "fp64 (DFMA/DMMA)", "kernel": dom,
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak,
                         "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                         "traffic_detail": traffic,
                         "work_model": "SURVEY 8(d) dense contractions (FMA = 2)",
                         "achieved_executed": dom_fx / (dom_ms * 1e-3) / 1e12,
                         "frac_executed": dom_fx / (dom_ms * 1e-3) / 1e12 / peak,
                         "even_odd": eo,
                         "peak_source": peak_src,
                         "step_frac": step_roof_ms / ms_step,
                         "step_frac_executed": max(fx_step / (peak * 1e12),
                                                   bytes_step / (hbm * 1e9)) * 1e3 / ms_step,
                         "step_flops_executed": fx_step,
                         "ncu_pipes": ncu_pipes,
                         "step_flops": flops_step, "step_bytes": bytes_step,
                         "hbm_peak_gbs": hbm, "hbm_source": hbm_src,
                         "kernel_ms": kt},
            "cpu_baseline": cpu,
            "determinism": ("AVS: the patch updates of a DoF are summed by fp64 bulk reduce-adds "
                            "in arbitrary order (run-to-run differences ~1e-16 relative); "
                            "DGB_AVS_ATOMIC=0 runs the deterministic colour order"
                            if kind == "avs" and os.environ.get("DGB_AVS_ATOMIC", "1") != "0"
                            else "deterministic launch order"),
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if slab:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 50; 3 for --impl reference)")
    ap.add_argument("--warmup", type=int, default=None,
                    help="untimed warm-up steps (default 5; 1 for --impl reference)")
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--slab", action="store_true",
                    help="run the multi-GPU slab code path even on one GPU (validation)")
    args = ap.parse_args()
    ref = args.impl == "reference"
    if args.steps is None:
        args.steps = 3 if ref else 50
    if args.warmup is None:
        args.warmup = 1 if ref else 5
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
