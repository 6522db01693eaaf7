#!/usr/bin/env python
"""Benchmark: full adaptive flow solve (frames -> u1, u2, mt with all alpha passes) in
Mpixel/s, fp64, on the B200 path; plus the HBM roofline of the dominant kernel (the
band forward/backward solve of the Schwarz preconditioner) and the CPU reference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

One step = one run_on_frames over one synthetic frame pair of the configuration (all
n_passes alpha updates and n_passes+1 converged Schwarz-PCG solves). ``value`` is timed
with CUDA events on the launching stream with frames already in HBM; ``e2e`` goes through
the host API (host frames in, u3 + alpha out). For N > 1 (torchrun) the subdomains of the one
frame pair are sharded over the ranks (strong scaling, paper_1508_02977_b200/parallel.py)
and the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full flow solve Mpixel/s (fp64)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    # c4 (2160x3840, 16x16 subdomains): the largest configuration, the one the north_star's
    # targets are quoted on; it fits one B200 (45 GB of factors)
    ap.add_argument("--config", default=os.environ.get("FFB_BENCH_CONFIG", "c4"))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # f64 (default, the headline): the preconditioner streams the subdomain factors in double.
    # f32: the opt-in single-precision COPY of the factors (ffb_set_factor_storage; the
    # factorisation, products, CG vectors and the stopping test stay in double, same 1e-8
    # parity) as the measured arm. The default run also reports it, separately, under
    # "variant_f32_factor_copy" unless --no-variants.
    ap.add_argument("--factor-storage", default="f64", choices=["f64", "f32"])
    ap.add_argument("--no-variants", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profiled_traffic(config):
    """dram bytes per launch of the band-solve kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "asm_traffic.json")) as fh:
            d = json.load(fh)
        return d.get(config)
    except Exception:
        return None


def run_config_for(cfg, ff):
    return ff.RunConfig(sigma=cfg.sigma, rho=cfg.rho, alpha0=cfg.alpha0, lambda0=cfg.lambda0,
                        parts=cfg.parts, overlap=cfg.overlap, adapt_iters=cfg.n_passes,
                        kappa=cfg.kappa, eta_threshold=cfg.eta_threshold,
                        cg_tolerance=cfg.tol)


def workload_config(cfg):
    """The `config` block of both arms' lines: the workload only (identical in both)."""
    from paper_1508_02977_b200 import flowfem as ff
    sp = ff.choose_split(cfg.W, cfg.H, cfg.parts)  # host-only (schwarz.cpp:32-44)
    px, py = sp.parts_x, sp.parts_y
    return {"workload": cfg.name, "H": cfg.H, "W": cfg.W, "parts": f"{px}x{py}",
            "overlap": cfg.overlap, "n_passes": cfg.n_passes, "tol": cfg.tol,
            "protocol": "converged-pass (SURVEY D2): n_passes x {solve to tol, "
                        "error_indicator, update_alpha} + final solve",
            "l2": "GPU arm: flushed (256 MB write) between steps; band factors > L2"}


def ref_iters(cfg):
    """Per-solve CG iteration counts of a full reference chain at the config's tolerance
    (tests/golden/ref_chain_iters.json, made by tests/golden/make_golden_large.py --iters)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "ref_chain_iters.json")) as fh:
            return json.load(fh).get(cfg.name)
    except Exception:
        return None


def cpu_reference_step(f0, f1, cfg):
    """One bounded step of the reference's own CPU path (oracle/_ref; the C port when the
    reference was not built), converged-pass protocol, all host cores. Configurations whose
    full chain is short (c1, c2) run it whole; the others run one timed instance of every
    stage (ref_chain_sample: imaging, mesh, assemble, CG set-up + iterations, indicator +
    update) and extrapolate the chain with the per-solve iteration counts of a committed full
    reference run. Returns (seconds, kind, cores, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    o = pyoracle.REF or pyoracle.PORT
    cores = os.cpu_count() or 1
    o.set_threads(cores)
    it = ref_iters(cfg)
    full = it is None or o is not pyoracle.REF or it["seconds"] * it["threads"] / cores <= 20.0
    if full:
        t = time.perf_counter()
        o.converged_chain(f0, f1, cfg.sigma, rho=cfg.rho, alpha0=cfg.alpha0, lambda0=cfg.lambda0,
                          n_passes=cfg.n_passes, kappa=cfg.kappa, thr=cfg.eta_threshold,
                          tol=cfg.tol)
        dt = time.perf_counter() - t
        return dt, o.kind, cores, (f"full converged-pass chain of {cfg.name} ({dt:.1f} s; "
                                   f"reference Jacobi-CG, monolithic), {cpu_model()}")
    smp = pyoracle.ref_chain_sample(f0, f1, cfg.sigma, rho=cfg.rho, alpha0=cfg.alpha0,
                                    lambda0=cfg.lambda0, kappa=cfg.kappa, thr=cfg.eta_threshold)
    dt = pyoracle.extrapolate_chain(smp, it["iters"])
    return dt, o.kind, cores, (
        f"extrapolated: one timed instance of every stage of the {cfg.name} chain on the real "
        f"input ({smp['wall']:.1f} s: imaging {smp['imaging']:.2f}, assemble {smp['assemble']:.2f}, "
        f"CG {smp['cg_iter'] * 1e3:.1f} ms/iteration, indicator+update {smp['adapt']:.2f} s) x the "
        f"{sum(it['iters'])} CG iterations of {len(it['iters'])} solves of a full reference run "
        f"(tests/golden/ref_chain_iters.json) = {dt:.1f} s per chain; {cpu_model()}")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def bench_reference(args, cfg, f0, f1):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    npx = cfg.H * cfg.W
    for _ in range(args.warmup):
        cpu_reference_step(f0, f1, cfg)
    times = []
    kind = cores = sample = None
    for _ in range(args.steps):
        dt, kind, cores, sample = cpu_reference_step(f0, f1, cfg)
        times.append(dt)
    tot = sum(times)
    v = npx * len(times) / tot / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "Mpixel/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg),
        "cpu_baseline": {"value": v, "unit": "Mpixel/s", "cores": cores, "kind": kind,
                         "sample": f"each step: {sample}"},
        "e2e": {"value": v, "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def fp64_peak():
    """FP64 denominator of the factor's roofline: profiles/fp64_peak.json (tools/microbench/
    fp64_peak.cu on the B200: device-wide DMMA rate), else the nominal DMMA rate."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            return float(json.load(fh)["dmma_tflops"]), "measured (profiles/fp64_peak.json)"
    except Exception:
        return 2 * 64 * 148 * 1.965e9 / 1e12, "nominal (64 DMMA FMA/clk/SM x 148 SMs x 1.965 GHz)"


def roofline_factor(s):
    """Second roofline: the subdomain factorisation (k_line_factor) against the FP64 tensor
    (DMMA) rate — algorithmic flops of one full factorisation (sum_i n_i kd_i^2, 2 flops per
    FMA) over the first pass's factorisation time (CUDA events on the launching stream; the
    later passes refactor incrementally)."""
    if not s.ms_factor_full or not s.factor_flops:
        return None
    peak, kind = fp64_peak()
    ach = s.factor_flops / (s.ms_factor_full * 1e-3) / 1e12
    return {"bound": "fp64 tensor (DMMA)", "kernel": "k_line_factor (full factorisation)",
            "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "peak_kind": kind, "flops_per_launch": s.factor_flops,
            "ms_per_launch": s.ms_factor_full, "traffic": None}


def maybe_spawn(args):
    """`bench.py --gpus N` without torchrun: launch the N ranks ourselves (one per GPU) through
    torch.distributed.run on 127.0.0.1, then exit with its status."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} GPUs, "
                                                     f"found {have}"}), flush=True)
        sys.exit(2)
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    maybe_spawn(args)
    rank, world, local = dist_env()
    from paper_1508_02977_b200 import synth
    f0, f1, _, cfg = synth.make(args.config, seed=0)
    if args.impl == "reference":
        bench_reference(args, cfg, f0, f1)
        return

    import numpy as np
    import torch
    from paper_1508_02977_b200 import flowfem as ff

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    ctx = ff.Context(local)
    stream = torch.cuda.Stream(dev)  # the launching stream: library kernels + timing events
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    if args.factor_storage == "f32":
        ctx.set_factor_storage(32)
    rc = run_config_for(cfg, ff)
    H, W = cfg.H, cfg.W
    npx = H * W
    d_f0 = torch.from_numpy(f0).to(dev)
    d_f1 = torch.from_numpy(f1).to(dev)
    d_u3 = torch.empty((3, H, W), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > L2

    if world > 1:
        # strong scaling: one frame pair; rank r owns a band of subdomain rows, the library
        # exchanges the overlap halos with its neighbours over NCCL P2P and all-reduces the CG
        # reduction units (parallel.py) — the same one call per step as N = 1
        from paper_1508_02977_b200 import parallel as par
        par.init_nccl(ctx, rank, world)

    def step():
        return ff.run_on_frames_device(d_f0.data_ptr(), d_f1.data_ptr(), W, H,
                                       d_u3.data_ptr(), rc, ctx)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ff.kernel_launches()
    stats = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))  # evict L2 between steps
            ev0[k].record(stream)
            stats.append(step())
            ev1[k].record(stream)
        torch.cuda.synchronize()
    launches = ff.kernel_launches() - launches0
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    tot_ms = sum(step_ms)
    if pg:
        t = torch.tensor([tot_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = npx * args.steps / (tot_ms / 1e3) / 1e6  # one frame pair per step (strong scaling)

    # end to end through the host API (pinned host frames in, u3 + alpha out)
    pin0 = torch.from_numpy(f0).pin_memory().numpy()
    pin1 = torch.from_numpy(f1).pin_memory().numpy()
    ctx.set_stream(None)

    def e2e_call():
        ff.run_on_frames(pin0, pin1, rc, ctx)
    e2e_call()  # warm
    e2e_times = []
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        if pg:
            pg.barrier()
        t0 = time.perf_counter()
        e2e_call()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_times) / len(e2e_times)
    if pg:
        t = torch.tensor([e2e_s], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": npx / e2e_s / 1e6, "unit": "Mpixel/s",
           "h2d_bytes_per_step": 2 * npx * 8,
           "d2h_bytes_per_step": 3 * npx * 8 + 2 * (W - 1) * (H - 1) * 8,
           "timing": "host wall clock around the blocking host-API call (max over ranks)"}

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return
    s = stats[-1]
    peak, peak_kind = measured_peak()
    f32_in_use = ctx.factor_storage()[1] == 32
    # packed line inverses, forward + backward sweep (4 bytes each from the opt-in f32 copy)
    asm_bytes = (4.0 if f32_in_use else 8.0) * s.factor_doubles
    try:
        from paper_1508_02977_b200 import _lib
        fn = _lib.load().ffb_debug_solve_kernel
        fn.restype, fn.argtypes = ctypes.c_int, [ctypes.c_void_p]
        kind = fn(ctx.handle)
    except Exception:
        kind = -1
    kname = {1: "k_line_solve_tile", 2: "k_line_solve_rt", 0: "k_line_solve"}.get(kind, "k_line_solve*")
    achieved = asm_bytes / (s.ms_asm_per_iter * 1e-3) / 1e9 if s.ms_asm_per_iter > 0 else None
    iters_total = s.pcg_iterations
    line = {
        "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(workload_config(cfg), factor_storage="f32 copy streamed by the solve "
                       "(factorisation, products, CG in f64)") if f32_in_use else workload_config(cfg),
        "parallelism": (f"row bands of subdomains over {world} GPUs, NCCL P2P halos + "
                        f"all-reduced CG units (bitwise equal to 1 GPU)") if world > 1 else "1gpu",
        "gpu_launches": int(launches),
        "e2e": e2e,
        "roofline": {"bound": "hbm", "kernel": f"{kname} (subdomain fwd/bwd sweeps)",
                     "unit_of_work": "one preconditioner application = forward + backward "
                                     "sweep launch (bytes_per_launch / ms_per_launch are per "
                                     "application)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": profiled_traffic(cfg.name), "peak_kind": peak_kind,
                     "bytes_per_launch": asm_bytes, "ms_per_launch": s.ms_asm_per_iter},
        "roofline_factor": roofline_factor(s),
        "solver": {"pcg_iterations_per_step": iters_total, "iters": s.iters,
                   "ms_terms": s.ms_terms, "ms_factor": s.ms_factor, "ms_pcg": s.ms_pcg,
                   "ms_adapt": s.ms_adapt, "ms_total": s.ms_total,
                   "iter_bytes": s.iter_bytes,
                   "pcg_iter_gbs": (s.iter_bytes * iters_total / (s.ms_pcg * 1e-3) / 1e9)
                   if s.ms_pcg > 0 else None},
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_variants and not f32_in_use:
        # Reported beside the headline, never as it: the same step with the solve kernel streaming
        # a single-precision copy of the subdomain factors (half the bytes per application;
        # everything else in double, same parity bar — tests/test_gpu_fullsize.py)
        try:
            variant_f32(ctx, stream, step, flush, torch, npx, args, line)
        except Exception as e:  # the headline line is printed whatever happens to the extra arm
            line["variant_f32_factor_copy"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if world == 1 and not args.no_cpu_baseline:
        dt, kind, cores, sample = cpu_reference_step(f0, f1, cfg)
        line["cpu_baseline"] = {"value": npx / dt / 1e6, "unit": "Mpixel/s", "cores": cores,
                                "kind": kind, "sample": sample}
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


def variant_f32(ctx, stream, step, flush, torch, npx, args, line):
    """The same step with the solve kernel streaming the single-precision factor copy (see the
    caller); leaves the context on double factors and its own stream."""
    ctx.set_stream(stream.cuda_stream)
    ctx.set_factor_storage(32)
    if ctx.factor_storage()[1] == 32:
        step()
        torch.cuda.synchronize()
        va, vb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nv = max(1, min(args.steps, 2))
        vstats = None
        flush.fill_(0.5)
        va.record(stream)
        for _ in range(nv):
            vstats = step()
        vb.record(stream)
        torch.cuda.synchronize()
        vms = va.elapsed_time(vb) / nv
        line["variant_f32_factor_copy"] = {
            "what": "opt-in ffb_set_factor_storage(32): the subdomain solve streams a "
                    "single-precision copy of the line inverses; factorisation, products, CG "
                    "vectors and the true-residual stopping test in f64; u within 1e-8 of the "
                    "reference like the default (not the headline, which stores doubles)",
            "value": npx / (vms * 1e-3) / 1e6, "unit": "Mpixel/s", "ms_per_step": vms,
            "steps": nv, "pcg_iterations_per_step": vstats.pcg_iterations,
            "ms_pcg": vstats.ms_pcg, "ms_factor": vstats.ms_factor,
            "solve_ms_per_application": vstats.ms_asm_per_iter,
            "solve_gbs": (4.0 * vstats.factor_doubles / (vstats.ms_asm_per_iter * 1e-3) / 1e9)
            if vstats.ms_asm_per_iter > 0 else None}
    ctx.set_factor_storage(64)
    ctx.set_stream(None)


if __name__ == "__main__":
    main()
