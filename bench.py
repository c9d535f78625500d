"""MHAR chain-step throughput on B200 (BASELINE.json metric).

A "step" is one iterate of every walk on every rank (the reference's
step(), proj/src/sampler.cpp:235-272), so

    value = walks_total x K / max-over-ranks device time   [chain-steps/s]

on the largest single-GPU BASELINE configuration: config 5, n = 2000,
m_I = 200000 unit-norm Gaussian rows, 4096 walks per GPU, fp64.  The
polytope (3.2 GB) is larger than L2, so no explicit flush is needed.

Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under
torch.distributed.run (one rank per GPU, NCCL).  --impl reference times the
CPU restatement of the reference (oracle/, the reference itself cannot be
built here) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")
METRIC = "MHAR chain-steps/sec at n=2000,m_I=2e5 fp64"


def fp64_peak():
    """Measured fp64 DMMA peak (tools/microbench_fp64.cu on this pool's
    B200; MEASURED_PEAKS.json carries no fp64 entry)."""
    best = None
    with open(PEAKS_FILE) as f:
        for line in f:
            d = json.loads(line)
            for k, v in d.items():
                if k.startswith("dmma_") and k.endswith("_tflops"):
                    best = v if best is None else max(best, v)
    return best


def _latest_ncu_file():
    """The newest committed `ncu --set full` summary (profiles/ncu_full_rNN.json)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_full_r*.json")))
    return files[-1] if files else os.path.join(ROOT, "profiles", "ncu_full_r01.json")


NCU_FILE = _latest_ncu_file()


def ncu_source() -> str:
    """Where roofline.traffic comes from: the capture file and, when it
    records them, the capture date and the commit of the captured kernels
    (traffic is not measured inside this run: ncu replays each kernel)."""
    name = os.path.relpath(NCU_FILE, ROOT)
    try:
        with open(NCU_FILE) as f:
            meta = json.load(f).get("_meta", {})
    except (OSError, ValueError):
        meta = {}
    if meta:
        return f"{name} (captured {meta.get('captured', '?')}, kernels at {meta.get('commit', '?')})"
    return f"{name} (round-1 capture, kernels of that round)"


def ncu_traffic(capture: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, GB)
    of the dominant kernel from the committed `ncu --set full` capture
    (tools/ncu_capture.sh), or None."""
    try:
        with open(NCU_FILE) as f:
            d = json.load(f)[capture]
        scale = {"Gbyte": 1.0, "Mbyte": 1e-3, "Tbyte": 1e3}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k]["value"]) * scale[d[k]["unit"]]
        return tot
    except (OSError, KeyError, ValueError):
        return None


I8_MMAS_PER_KSTEP = 34  # slice-pair products per k step (chord_i8.cuh)


TENSOR_PROBE = os.path.join(ROOT, "profiles", "tensor_probe_r01.jsonl")


def _probe_peak(key: str):
    """Best rate of the MMA-only tcgen05 microbenchmark (tools/i8_probe.cu on
    this pool's B200, profiles/tensor_probe_r01.jsonl) for `key`."""
    best = None
    try:
        with open(TENSOR_PROBE) as f:
            for line in f:
                v = json.loads(line).get(key)
                if v is not None:
                    best = v if best is None else max(best, v)
    except (OSError, ValueError):
        pass
    return best


def int8_dense_peak():
    """Dense int8 tensor-core peak (tcgen05 kind::i8 microbench); fallback
    4500 TOPS (nominal)."""
    return _probe_peak("int8_tops") or 4500.0


def tf32_dense_peak():
    """TF32 tensor-core peak: the tcgen05 kind::tf32 microbench (CTA pair,
    N = 256, the fp32 variant's shape); fallback the driver-measured dense
    bf16 GEMM rate halved (MEASURED_PEAKS.json), then 1590/2."""
    v = _probe_peak("tf32_tflops")
    if v:
        return v
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["bf16_tflops"] / 2.0
    except (OSError, KeyError, ValueError):
        return 1590.0 / 2.0


def measured_bf16_peak():
    """Dense bf16 TFLOP/s from the driver-written MEASURED_PEAKS.json (burst:
    the fp32 variant's kernel is timed in a short region), or None."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return None


def f16_probe_peak():
    """kind::f16 MMA-only microbench (tools/i8_probe.cu, CTA pair, N = 256),
    the stricter figure reported beside the prescribed peak."""
    return _probe_peak("f16_tflops") or 2250.0


def f16_dense_peak():
    """FP16 (f32 accumulate) tensor-core roofline: the driver-measured dense
    bf16 peak in MEASURED_PEAKS.json (kind::f16 and kind::bf16 run at the same
    rate); fallback the MMA-only microbench."""
    return measured_bf16_peak() or f16_probe_peak()


def tc_form():
    """Form of the fp32 variant's kernel: "f16" (default) or "tf32" (MHAR_TC_F16=0)."""
    return "tf32" if os.environ.get("MHAR_TC_F16", "1") == "0" else "f16"


def tc_roofline_terms():
    """(peak, unit, kernel, dtype, peak source) of the fp32 variant's form."""
    if tc_form() == "f16":
        return (f16_dense_peak(), "TFLOP/s (F16 executed)",
                "chord_tc32_kernel<F16> (tcgen05.mma kind::f16, TMEM, bulk-copy ring)",
                "A_I as two fp16 halves per row scale (22 bits of the row maximum); products "
                "exact, f32 accumulate; slack and walks f64",
                "MEASURED_PEAKS.json bf16_tflops (driver-measured dense bf16, burst)"
                if measured_bf16_peak() else
                "tcgen05 kind::f16 microbench, profiles/tensor_probe_r01.jsonl")
    return (tf32_dense_peak(), "TFLOP/s (TF32 executed)",
            "chord_tc32_kernel (tcgen05.mma kind::tf32, TMEM, bulk-copy ring)",
            "A_I rounded to f32; rates f32-accurate on tcgen05 (TF32 hi/lo split); "
            "slack and walks f64",
            "tcgen05 kind::tf32 microbench, profiles/tensor_probe_r01.jsonl")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.out = out
        else:
            self.out = ""

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for line in self.out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    """One process per GPU, NCCL.  MHAR_SHARE_GPU=1 (functional testing of
    the multi-rank path on a one-GPU box only) maps every rank to device 0
    and runs the collectives on gloo; such timings are not bench numbers."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("MHAR_SHARE_GPU") == "1":
            local = 0
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def coll_device():
    """Device for collective tensors: CUDA under NCCL, CPU under gloo."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_backend() == "gloo":
        return "cpu"
    return "cuda"


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_model() -> str:
    """Host CPU model name (state the CPU beside the core count)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(w, z_sample: int, iters: int, threads: int):
    """The oracle (CPU restatement of the reference step) on a bounded
    sample of the same workload: z_sample walks x iters iterates."""
    import oracle
    L = oracle.lib()
    L.orc_set_threads(threads)
    p = w.polytope
    X = np.zeros((p.dim(), z_sample), order="F")
    X[:] = w.x0[:, None]
    rng = oracle.WalkRng(1234, z_sample)
    P = None
    if p.num_equalities():
        st, P, _ = oracle.compute_projection(p.a_eq)
    st, _, _ = oracle.step(p.a_in, p.b_in, P, 1e-11, rng, X)  # warm-up
    t0 = time.perf_counter()
    for _ in range(iters):
        st, _, _ = oracle.step(p.a_in, p.b_in, P, 1e-11, rng, X)
        assert st == 0
    dt = time.perf_counter() - t0
    return z_sample * iters / dt, dt


def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_2104_07097_b200 import workloads
    import oracle
    w = workloads.config(args.config, z=args.z)
    threads = os.cpu_count() or 1
    oracle.lib().orc_set_threads(threads)
    p = w.polytope
    X = np.zeros((p.dim(), args.cpu_walks), order="F")
    X[:] = w.x0[:, None]
    rng = oracle.WalkRng(args.seed, args.cpu_walks)
    P = oracle.compute_projection(p.a_eq)[1] if p.num_equalities() else None
    for _ in range(args.warmup):
        assert oracle.step(p.a_in, p.b_in, P, 1e-11, rng, X)[0] == 0
    total = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        assert oracle.step(p.a_in, p.b_in, P, 1e-11, rng, X)[0] == 0
        total += time.perf_counter() - t0
    value = args.cpu_walks * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "chain-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * args.cpu_walks / value, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n": w.polytope.dim(), "m_I": w.polytope.num_inequalities(),
                   "m_E": w.polytope.num_equalities(), "walks_per_step": args.cpu_walks},
        "cpu_baseline": {"value": value, "unit": "chain-steps/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.cpu_walks} walks x 1 iterate per step of the config-"
                                   f"{args.config} polytope (oracle/mhar_oracle.c, OpenMP GEMM)"},
        "e2e": {"value": value, "unit": "chain-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# The paper's published MHAR throughputs (fp64,
# best padding z* per body/dimension): (figure, n, z*, samples/s).
PAPER_TABLE = [
    ("hypercube", 3, 10000, 25357073.87), ("hypercube", 5, 10000, 13206089.93),
    ("hypercube", 15, 10000, 25344794.68), ("hypercube", 25, 5000, 10839474.35),
    ("hypercube", 50, 2500, 5151516.81), ("hypercube", 100, 4000, 4363525.70),
    ("hypercube", 250, 3000, 1219419.53), ("hypercube", 500, 4000, 621554.24),
    ("hypercube", 1000, 4000, 248513.69), ("hypercube", 2500, 1500, 50808.74),
    ("hypercube", 5000, 1000, 16161.69),
    ("simplex", 3, 10000, 19795014.21), ("simplex", 5, 10000, 22878783.33),
    ("simplex", 15, 10000, 24269548.32), ("simplex", 25, 10000, 24338761.06),
    ("simplex", 50, 10000, 13425900.57), ("simplex", 100, 3000, 7255837.08),
    ("simplex", 250, 4000, 2656449.22), ("simplex", 500, 1500, 944784.52),
    ("simplex", 1000, 500, 329315.49), ("simplex", 2500, 500, 77312.01),
    ("simplex", 5000, 1000, 22437.63),
]


def run_paper(args):
    """The paper's own benchmark (Avg. samples/s = z phi T / Time,
    PAPER.md:694-698) on its bodies and padding z*, through run() on one
    B200: phi is sized so each run takes ~0.5 s (the paper used 30,000)."""
    import paper_2104_07097_b200 as mh
    out = []
    for fig, n, z, paper in PAPER_TABLE:
        if fig == "hypercube":
            p, x0 = mh.make_hypercube(n), np.zeros(n)
        else:
            p, x0 = mh.make_simplex(n), np.full(n, 1.0 / n)
        proj = mh.compute_projection(p.a_eq) if p.num_equalities() else None
        with mh.Engine(p, z, seed=args.seed, projector=proj) as eng:
            _, st = eng.run(x0, 20, 1, 0, 20 if proj else 0)  # warm-up + cost probe
            per_iter = st.seconds / 20
            phi = int(min(30000, max(50, 0.5 / max(per_iter, 1e-9))))
            _, st = eng.run(x0, phi, 1, 0, phi if proj else 0)
        value = z * phi / st.seconds
        rec = {"figure": fig, "n": n, "z": z, "phi": phi, "seconds": st.seconds,
               "chain_steps_per_s": value, "paper_p100": paper, "ratio_vs_paper": value / paper}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    return out


def run_sweep(args):
    """Padding sweep (the reference's sweep_padding, proj/src/bench.cpp:49-61,
    and the paper's z* experiment): chain-steps/s against
    the walk count z on one B200, phi and the body fixed.  The paper
    conjectured that large z causes memory contention on its P100."""
    import paper_2104_07097_b200 as mh
    from paper_2104_07097_b200 import workloads
    w = workloads.config(args.config)
    p = w.polytope
    proj = mh.compute_projection(p.a_eq) if p.num_equalities() else None
    out = []
    for z in [int(v) for v in args.sweep_z.split(",")]:
        for prec in ([64, 32] if args.config >= 3 else [64]):
            with mh.Engine(p, z, seed=args.seed, projector=proj, precision=prec) as eng:
                X = np.empty((p.dim(), z), order="F")
                X[:] = w.x0[:, None]
                eng.set_state(X)
                eng.step_timed(3, 0)
                ms = eng.step_timed(args.steps, 0)
            rec = {"sweep": "padding", "config": args.config, "precision": prec, "z": z,
                   "chain_steps_per_s": z * args.steps / (ms * 1e-3),
                   "ms_per_iterate": ms / args.steps}
            out.append(rec)
            print(json.dumps(rec), flush=True)
    return out


def timed_cycle(eng, steps: int, reproject: int, refresh_every: int, incremental: bool,
                world: int, clock_device=None):
    """The timed region of one engine: a refresh pass (the fresh fused / A x
    product that rebuilds the incremental slack cache) followed by steps - 1
    incremental iterates, each part bracketed by CUDA events on the engine's
    stream.  Returns the refresh-amortized device time per iterate,
    (t_refresh + (R - 1) t_incremental) / R with R = refresh_every -- the
    long-run cost of an iterate in a run() -- plus the per-part stats of the
    chord kernels and the clocks sampled during the region."""
    eng.request_refresh()
    eng.reset_stats()
    eng.set_timing(True)
    barrier(world)
    clk = ClockSampler(clock_device) if clock_device is not None else None
    if clk:
        clk.__enter__()
    ms_ref = eng.step_timed(1, reproject)
    s_ref = eng.stats()
    eng.reset_stats()
    ms_rest = eng.step_timed(max(steps - 1, 1), reproject)
    if clk:
        clk.__exit__(None, None, None)
    eng.set_timing(False)
    s_rest = eng.stats()
    ms_ref = max_over_ranks(ms_ref, world)
    ms_rest = max_over_ranks(ms_rest, world)
    t_inc = ms_rest / max(steps - 1, 1)
    if incremental:
        amortized = (ms_ref + (refresh_every - 1) * t_inc) / refresh_every
    else:
        amortized = (ms_ref + ms_rest) / (1 + max(steps - 1, 1))
    return {"ms_per_iterate": amortized, "ms_refresh": ms_ref, "ms_incremental": t_inc,
            "ms_region": ms_ref + ms_rest, "stats_refresh": s_ref, "stats": s_rest,
            "launches": s_ref["kernel_launches"] + s_rest["kernel_launches"],
            "clocks": clk.summary() if clk else None}


def run_group(args):
    """--driver group: one process drives --gpus N devices through the C
    ABI's multi-device group (mhar_group_*; one host thread and stream per
    device, walks sharded by global id, windows gathered to device 0 over
    NCCL).  Same workload per device as the torchrun path; the timed region
    is a group step of K iterates bracketed by a host clock after a device
    sync on every GPU (the group step returns only when all shards are done),
    and the chord kernels' CUDA-event times per device are reported beside."""
    import paper_2104_07097_b200 as mh
    from paper_2104_07097_b200 import workloads
    import torch
    ndev = args.gpus
    devices = list(range(ndev)) if torch.cuda.device_count() >= ndev else [0] * ndev
    w = workloads.config(args.config, z=args.z)
    p = w.polytope
    z_total = w.z * ndev
    projector = mh.compute_projection(p.a_eq) if p.num_equalities() else None
    reproject = args.reproject if p.num_equalities() else 0
    g = mh.Group(p, z_total, devices, seed=args.seed, projector=projector,
                 refresh_every=args.refresh)
    X0 = np.empty((p.dim(), z_total), order="F")
    X0[:] = w.x0[:, None]
    g.set_state(X0)
    g.step(args.warmup, reproject)
    t0 = time.perf_counter()
    g.step(args.steps, reproject)
    secs = time.perf_counter() - t0
    value = z_total * args.steps / secs
    # one collection window through run(): rows of every shard on device 0,
    # then on the host (the samples of a window, 65.5 MB per shard at config 5)
    t1 = time.perf_counter()
    S, st = g.run(w.x0, phi=args.steps, windows=1, burn_in=0, reproject_every=reproject)
    run_s = time.perf_counter() - t1
    info = g.info()
    g.close()
    line = {"metric": METRIC, "value": value, "unit": "chain-steps/s", "n_gpus": ndev,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded unit-norm Gaussian rows, BASELINE config %d)" % args.config,
            "config": {"workload": w.name, "walks_per_gpu": w.z, "walks_total": z_total,
                       "driver": "mhar_group (one process, one thread per device)",
                       "devices": devices, "uses_nccl": info["uses_nccl"]},
            "timing": "host clock around a group step that synchronises every device",
            "run_one_window": {"value": z_total * args.steps / run_s, "seconds": run_s,
                               "samples_rows": int(S.shape[0]),
                               "max_violation": info["last_max_violation"]}}
    print(json.dumps(line), flush=True)


def run_engine(args, world, rank, local):
    import paper_2104_07097_b200 as mh
    from paper_2104_07097_b200 import workloads

    offset = None
    if args.strong:
        # strong scaling: a fixed job of --strong walks split
        # into contiguous per-rank ranges keyed on the global chain id
        base, extra = divmod(args.strong, world)
        z_local = base + (1 if rank < extra else 0)
        offset = rank * base + min(rank, extra)
        w = workloads.config(args.config, z=z_local)
    else:
        w = workloads.config(args.config, z=args.z)
    p = w.polytope
    z = w.z
    total_walks = args.strong if args.strong else z * world
    if offset is None:
        offset = rank * z
    # the committed ncu captures (NCU_FILE) are of this workload
    captured = args.config == 5 and z == 4096
    traffic = {k: ncu_traffic(k) for k in ("chord2_full", "chord3_full", "tc32_full", "tc32r_full",
                                           "i8_full")}
    traffic_source = ncu_source()
    projector = mh.compute_projection(p.a_eq) if p.num_equalities() else None
    reproject = args.reproject if p.num_equalities() else 0
    eng = mh.Engine(p, z, seed=args.seed, projector=projector, slack=args.slack,
                    refresh_every=args.refresh, device=local, chain_offset=offset,
                    precision=args.precision, f64_engine=args.f64_engine,
                    fp32_direction=args.fp32_direction, z_plan=total_walks)
    X0 = np.zeros((p.dim(), z), order="F")
    X0[:] = w.x0[:, None]
    eng.set_state(X0)

    # warm-up; the first iterate after set_state is the fused refresh pass
    # (A_I [X | D] + slack cache), which recurs every --refresh iterates
    eng.step_timed(args.warmup, reproject)

    # timed, device-resident inputs: one refresh pass + K - 1 incremental
    # iterates; value is the refresh-amortized rate
    incremental = args.slack == "incremental"
    cyc = timed_cycle(eng, args.steps, reproject, args.refresh, incremental, world, local)
    st = cyc["stats"]
    ms = cyc["ms_per_iterate"] * args.steps
    value = total_walks / (cyc["ms_per_iterate"] * 1e-3)

    # e2e: the reference-facing call with HOST buffers every step, as the
    # reference's own loop `step(p, op, cfg, rng, state)` does: the walk state
    # goes host -> device (pinned), one iterate, device -> host.  Two forms:
    # the caller hands back the state unchanged (the reference's loop; the
    # slack cache survives) and the caller edits X before every step (each
    # step then pays the refresh pass).
    import torch
    pinned = torch.empty((z, p.dim()), dtype=torch.float64, pin_memory=True).numpy()
    Xh = pinned.T  # (n, z) column-major view of pinned memory
    eng.get_state(out=Xh)

    def e2e_loop(steps, mutate):
        barrier(world)
        t = 0.0
        for i in range(steps):
            if mutate:
                Xh[0, :] *= 1.0 - 1e-12  # an edit the cache cannot survive
            t0 = time.perf_counter()
            eng.set_state(Xh)
            eng.step(1, reproject)
            eng.get_state(out=Xh)
            t += time.perf_counter() - t0
        return max_over_ranks(t, world)

    e2e_s = e2e_loop(args.e2e_steps, False)
    e2e_value = total_walks * args.e2e_steps / e2e_s
    e2e_mut_steps = max(3, args.e2e_steps // 4)
    e2e_mut_s = e2e_loop(e2e_mut_steps, True)
    e2e_mut_value = total_walks * e2e_mut_steps / e2e_mut_s
    bytes_state = p.dim() * z * 8

    # one collection window (outside the timed region): containment of every
    # walk, rows gathered device-to-device to rank 0 and diagnostics reduced
    # -- the only collectives of a multi-GPU run (NCCL over NVLink).
    from paper_2104_07097_b200.distributed import gather_rows, reduce_diagnostics
    bad, viol, eqv = eng.check_state(eng.eps_feas)
    rows = torch.empty((z, p.dim()), dtype=torch.float64, device=f"cuda:{local}")
    eng.state_rows_to_device(rows.data_ptr())
    if coll_device() == "cpu":
        rows = rows.cpu()
    diag = reduce_diagnostics(st["redraw_count"], float(viol.max()), float(eqv.max()), rows,
                              device=rows.device)
    gathered = gather_rows(rows, [z] * world)

    fpi = eng.flops_per_iterate()
    chord_avg_ms = st["chord_ms"] / max(st["chord_timed"], 1)
    chord_kernel = st["chord_kernel"]  # chord3_kernel from n_pad >= 384, else chord2_kernel
    chord_capture = "chord3_full" if chord_kernel == "chord3_kernel" else "chord2_full"
    achieved = st["chord_flops"] / max(st["chord_ms"] * 1e-3, 1e-30) / 1e12
    peak = fp64_peak()
    eng.close()

    # the int8-slice fp64 engine (Ozaki scheme on the tcgen05 int8 tensor cores)
    # on the same workload: fp64-accurate rates, reported beside the DMMA line
    i8 = None
    if args.precision == 64 and not args.no_i8 and p.dim() <= 4608:
        e8 = mh.Engine(p, z, seed=args.seed, projector=projector, refresh_every=args.refresh,
                       device=local, chain_offset=rank * z, f64_engine="int8")
        e8.set_state(X0)
        e8.step_timed(args.warmup, reproject)
        c8 = timed_cycle(e8, args.steps, reproject, args.refresh, True, world)
        ms8 = c8["ms_per_iterate"] * args.steps
        s8 = c8["stats"]
        bad8, viol8, _ = e8.check_state(e8.eps_feas)
        e8.close()
        alg8 = s8["chord_flops"] / max(s8["chord_ms"] * 1e-3, 1e-30) / 1e12
        ops8 = I8_MMAS_PER_KSTEP * alg8  # int8 tensor ops executed (34 slice-pair products)
        i8_peak = int8_dense_peak()
        i8 = {"value": total_walks * args.steps / (ms8 * 1e-3), "unit": "chain-steps/s",
              "ms_per_step": ms8 / args.steps,
              "dtype": "f64 results: A_I and d as 53-bit fixed point in 7 int8 slices, exact "
                       "int32 slice products (levels 0..7), fp64 combine; slack and walks f64",
              "kernel": "chord_i8_kernel (tcgen05.mma kind::i8, CTA pair, 8 TMEM level accumulators)",
              "fp64_equivalent_tflops": alg8, "fp64_equivalent_frac_of_dmma_peak": alg8 / peak,
              "roofline": {"bound": "tensor", "achieved": ops8, "peak": i8_peak,
                           "unit": "TOPS (int8 executed)", "frac": ops8 / i8_peak,
                           "traffic": traffic["i8_full"] if captured else None,
                           "peak_source": "tcgen05 kind::i8 microbench, profiles/tensor_probe_r01.jsonl"},
              "all_inside_eps_feas": bool(bad8 == -1)}

    # the north star's fp32 variant on the same workload (A_I rounded to fp32,
    # rates on tcgen05 tensor cores): same timing protocol, reported beside
    def fp32_line(direction):
        """The north star's fp32 variant on the same workload, same timing
        protocol.  direction "split": the walk moves along its fp64
        direction, the tensor cores see it as two operands (3 MMAs per k
        step); "rounded": the fast form, the direction rounded to one
        operand and moved along (2 MMAs)."""
        e32 = mh.Engine(p, z, seed=args.seed, projector=projector, refresh_every=args.refresh,
                        device=local, chain_offset=rank * z, precision=32,
                        fp32_direction=direction)
        e32.set_state(X0)
        e32.step_timed(args.warmup, reproject)
        c32 = timed_cycle(e32, args.steps, reproject, args.refresh, True, world)
        s32 = c32["stats"]
        bad32, viol32, _ = e32.check_state(e32.eps_feas)
        e32.close()
        mmas = 3.0 if (direction == "split" or p.num_equalities()) else 2.0
        tc_exec = mmas * s32["chord_flops"] / max(s32["chord_ms"] * 1e-3, 1e-30) / 1e12
        tc_peak, tc_unit, tc_kernel, tc_dtype, tc_src = tc_roofline_terms()
        return {"value": total_walks / (c32["ms_per_iterate"] * 1e-3), "unit": "chain-steps/s",
                "ms_per_step": c32["ms_per_iterate"], "form": tc_form(), "direction": direction,
                "dtype": tc_dtype + ("; direction split into two operands, walk moves along "
                                     "its fp64 direction" if direction == "split" else
                                     "; direction rounded to one operand and moved along"),
                "kernel": tc_kernel, "mmas_per_kstep": mmas,
                "roofline": {"bound": "tensor", "achieved": tc_exec, "peak": tc_peak,
                             "unit": tc_unit, "frac": tc_exec / tc_peak,
                             "frac_vs_mma_probe": (tc_exec / f16_probe_peak()
                                                   if tc_form() == "f16" else None),
                             "traffic": (traffic["tc32_full" if direction == "split" else
                                                 "tc32r_full"] if captured else None),
                             "traffic_unit": "GB DRAM read+write per launch (ncu --set full)",
                             "avg_launch_ms": s32["chord_ms"] / max(s32["chord_timed"], 1),
                             "peak_source": tc_src},
                "all_inside_eps_feas": bool(bad32 == -1),
                "containment_body": "caller's fp64 A_I (fresh DMMA product)"}

    fp32 = fp32r = None
    if args.precision == 64 and not args.no_fp32:
        fp32 = fp32_line("split")
        fp32r = fp32_line("rounded")

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        v, dt = cpu_sample(w, args.cpu_walks, args.cpu_iters, threads)
        cpu = {"value": v, "unit": "chain-steps/s", "cores": threads, "kind": "port",
               "cpu_model": cpu_model(),
               "sample": f"{args.cpu_walks} walks x {args.cpu_iters} iterates of the same polytope "
                         f"({dt:.1f} s; oracle/mhar_oracle.c restating proj/src/sampler.cpp, "
                         f"OpenMP AVX-512 GEMM)"}
        if args.cpu_walks_1core > 0:
            # the reference itself is single-threaded (no OpenMP):
            # the same port on one core, smaller sample
            v1, dt1 = cpu_sample(w, args.cpu_walks_1core, args.cpu_iters_1core, 1)
            cpu["single_core"] = {
                "value": v1, "cores": 1,
                "sample": f"{args.cpu_walks_1core} walks x {args.cpu_iters_1core} iterates "
                          f"({dt1:.1f} s)"}
    line = {
        "metric": METRIC, "value": value, "unit": "chain-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded unit-norm Gaussian rows, BASELINE config %d)" % args.config,
        "config": {"workload": w.name, "n": p.dim(), "m_I": p.num_inequalities(),
                   "m_E": p.num_equalities(), "walks_per_gpu": z, "walks_total": total_walks,
                   "slack_mode": args.slack, "refresh_every": args.refresh, "rng": "philox",
                   "parallelism": f"walk-sharded x{world}",
                   "l2": "inputs larger than L2 (A_I is %.1f GB)" % (p.a_in.nbytes / 1e9)},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": traffic[chord_capture] if captured else None,
                     "traffic_unit": "GB DRAM read+write per launch (ncu --set full)",
                     "traffic_source": traffic_source,
                     "algorithmic_bytes_GB": (p.a_in.nbytes + 4 * 8 * z * p.num_inequalities()
                                              + 8 * z * p.dim()) / 1e9,
                     "kernel": (("chord3_kernel (DMMA A_I D, accumulators handed through TMEM "
                                 "to epilogue warps: streamed slack cache, fused chord reduce)")
                                if chord_kernel == "chord3_kernel" else
                                f"{chord_kernel}<INCREMENTAL> (DMMA A_I D + streamed slack cache, "
                                "fused chord reduce)"),
                     "avg_launch_ms": chord_avg_ms, "launches": st["chord_timed"],
                     "peak_source": "fp64 DMMA microbench, profiles/fp64_peaks_r01.json",
                     "peak_note": "builder-measured mma.sync.m8n8k4.f64 throughput on this pool's "
                                  "B200 (MEASURED_PEAKS.json has no fp64 entry; cuBLAS DGEMM "
                                  "reaches 35.5 TFLOP/s on the same box)"},
        "reference_equivalent_tflops": value * fpi / z / 1e12 / world,
        "refresh": {"every": args.refresh, "ms_refresh_pass": cyc["ms_refresh"],
                    "ms_incremental_iterate": cyc["ms_incremental"],
                    "steady_value": total_walks / (cyc["ms_incremental"] * 1e-3),
                    "note": "the timed region is one refresh pass + K-1 incremental iterates; "
                            "value = walks / ((t_refresh + (every-1) t_incremental) / every), the "
                            "long-run rate with one refresh per `every` iterates"},
        "e2e": {"value": e2e_value, "unit": "chain-steps/s", "h2d_bytes_per_step": bytes_state,
                "d2h_bytes_per_step": bytes_state, "steps": args.e2e_steps,
                "note": "host state in, one iterate, host state out per step (the reference's "
                        "step(p, op, cfg, rng, state) loop, state handed back unchanged)"},
        "e2e_mutated": {"value": e2e_mut_value, "unit": "chain-steps/s",
                        "h2d_bytes_per_step": bytes_state, "d2h_bytes_per_step": bytes_state,
                        "steps": e2e_mut_steps,
                        "note": "the host edits X before every step: each step pays the refresh "
                                "pass"},
        "gpu_launches": cyc["launches"],
        "clocks": cyc["clocks"],
        "checks": {"walks_gathered_on_rank0": int(gathered.shape[0]),
                   "max_violation": diag.max_violation, "max_eq_residual": diag.max_eq_residual,
                   "all_inside_eps_feas": bool(diag.max_violation <= 1e-9 and
                                               diag.max_eq_residual <= 1e-9),
                   "redraws": diag.redraws},
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if fp32:
        line["fp32_variant"] = fp32
    if fp32r:
        line["fp32_variant_rounded_direction"] = fp32r
    if i8:
        line["fp64_int8_variant"] = i8
    if args.precision == 32:
        tc_peak, tc_unit, tc_kernel, tc_dtype, tc_src = tc_roofline_terms()
        line["dtype"] = "f32 rates (" + tc_dtype + ")"
        mm = 3.0 if args.fp32_direction == "split" or p.num_equalities() else 2.0
        line["roofline"].update({"achieved": mm * achieved, "peak": tc_peak, "unit": tc_unit,
                                 "frac": mm * achieved / tc_peak, "kernel": tc_kernel,
                                 "traffic": traffic["tc32_full"] if captured else None,
                                 "peak_source": tc_src})
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--z", type=int, default=None)
    ap.add_argument("--strong", type=int, default=0,
                    help="strong scaling: a fixed total of this many walks split over the ranks")
    ap.add_argument("--seed", type=int, default=2021)
    ap.add_argument("--slack", default="incremental", choices=["incremental", "recompute"])
    ap.add_argument("--refresh", type=int, default=128)
    ap.add_argument("--reproject", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-walks", type=int, default=256)
    ap.add_argument("--cpu-iters", type=int, default=24)
    ap.add_argument("--cpu-walks-1core", type=int, default=32)
    ap.add_argument("--cpu-iters-1core", type=int, default=4)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32-variant measurement")
    ap.add_argument("--no-i8", action="store_true", help="skip the int8-slice fp64 engine")
    ap.add_argument("--f64-engine", default="dmma", choices=["dmma", "int8"],
                    help="engine of the headline fp64 line (default: DMMA)")
    ap.add_argument("--sweep-z", default="",
                    help="comma-separated walk counts: padding sweep instead of the bench line")
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32],
                    help="32: the fp32 variant (tcgen05 3xTF32 rates, fp64 state)")
    ap.add_argument("--fp32-direction", default="split", choices=["split", "rounded"],
                    help="--precision 32: split (default, north-star parity) or rounded "
                         "(fast form) direction")
    ap.add_argument("--driver", default="ranks", choices=["ranks", "group"],
                    help="ranks: one process per GPU (torchrun); group: this process drives "
                         "--gpus devices through the C ABI's mhar_group")
    ap.add_argument("--paper", action="store_true",
                    help="run the paper's hypercube/simplex table (PAPER.md:845-887) instead")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference" and not (args.paper or args.sweep_z):
        # CPU-only arm: rank 0 times the reference restatement, the other
        # ranks exit 0 without work; no process group, no device touched
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")),
                      int(os.environ.get("RANK", "0")))
        return
    if args.driver == "group":
        run_group(args)
        return
    world, rank, local = dist_setup(args)
    if args.paper:
        run_paper(args)
    elif args.sweep_z:
        run_sweep(args)
    else:
        run_engine(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
