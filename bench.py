"""Benchmark of the spatial-voting path (BASELINE.json metric) on 1..8 B200s.

Workload (BASELINE.json configs[2], the headline metric's config): estimate_single on
N = 1,000,000 correspondences, 90% outliers, sigma = 0.01 (synthetic, seeded).
One step = one full solve (preprocess, vote, peak, refine, angle vote, rotation).

  value  = correspondences/sec of the device-resident solve (inputs already in HBM), all ranks
  e2e    = the same through the public C-ABI with host buffers: pinned H2D of the 48 MB input
           and D2H of the estimate + inlier list inside the timed region
  e2e_pageable = the reference user's call: C++ rotavote::estimate_single on a fresh
           std::vector<Correspondence> (pageable memory), host clock (tools/e2e/e2e_pageable.cpp)
  roofline: dominant kernel = the band-tiled vote (K2), bound by shared-memory atomics/ALU;
           peak = conflict-free u32 shared-atomic rate measured live on this box
  cpu_baseline / cpu_baseline_1thread: the reference (oracle/_ref, unmodified sources, reference
           flags) on the host cores (cfg.threads = nproc, and the reference default 1), rank 0 at N=1

Multi-GPU (--gpus N: re-launches itself under torchrun when WORLD_SIZE is unset; --mode sharded,
default): one C3 problem, correspondences sharded across ranks, per-rank vote, NCCL all-reduce of
the uint32 grid, sharded refine_loop / angle vote with rank-ordered partial sums
(distributed.sharded_estimate_single; "scaling": "strong"); --mode replicas: one
independent problem per rank ("weak"). Device time = max over ranks. NCCL_DEBUG=INFO lines go to
stderr.
`--impl reference` runs the reference CPU implementation instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "correspondences/sec voted (axis+angle) at N=1e6, 90% outliers; ms per solve"
UNIT = "correspondences/s"
WORKLOAD = "c3"


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def config_block(n: int, world: int, extra: dict | None = None) -> dict:
    d = {"workload": "BASELINE configs[2]: estimate_single, N=1e6 correspondences, 90% outliers, sigma=0.01",
         "n_per_solve": n, "grid": 512, "extent": 1.05, "theta_samples": 2048, "epsilon": 0.015,
         "angle_bins": 1024, "solves_per_step": world,
         "parallelism": f"replicas{world}" if world > 1 else "single",
         "l2": "flushed between timed steps (256 MiB write; input 48 MB < 126 MB L2)"}
    if extra:
        d.update(extra)
    return d


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                pass
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def smem_atomic_peak(device: int):
    lib_path = ROOT / "tools" / "microbench" / "libsmem_atomics.so"
    if not lib_path.exists():
        return None
    lib = C.CDLL(str(lib_path))
    r, ms = C.c_double(), C.c_double()
    if lib.smem_atomic_peak(device, C.byref(r), C.byref(ms)) != 0:
        return None
    return r.value


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "fallback": True}


def vote_profile():
    """ncu --set full summary of the vote kernel committed under profiles/ (traffic, issue rate)."""
    for rnd in ("r2", "r1"):  # the latest committed capture
        p = ROOT / "profiles" / rnd / "vote_kernel_ncu.json"
        if p.exists():
            return json.loads(p.read_text())
    return None


def reference_cpu(n_sample: int, reps: int, threads: int, corrs: np.ndarray):
    """The reference's own estimate_single (oracle/_ref, -O3 -march=native) on the host cores."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc
    kind = "ref_perf"
    try:
        ref = orc.Oracle(kind)
    except (FileNotFoundError, OSError):
        kind = "port"
        ref = orc.Oracle(kind)
    cfg = orc.default_config(threads=threads)
    sample = np.ascontiguousarray(corrs[:n_sample])
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.estimate_single(sample, cfg)
        times.append(time.perf_counter() - t0)
    return kind, times


def pageable_e2e(corrs: np.ndarray, steps: int, warmup: int, d2h_bytes: int):
    """The reference user's path: rotavote::estimate_single (C++ drop-in, estimator.hpp:63-64) on a
    fresh std::vector<Correspondence> in pageable memory, host clock around the call
    (tools/e2e/e2e_pageable.cpp)."""
    import subprocess
    import tempfile
    exe = ROOT / "tools" / "_bin" / "e2e_pageable"
    if not exe.exists():
        return {"unavailable": "tools/_bin/e2e_pageable not built (tools/e2e: make)"}
    with tempfile.NamedTemporaryFile(suffix=".f64") as f:
        np.ascontiguousarray(corrs, dtype=np.float64).tofile(f.name)
        r = subprocess.run([str(exe), f.name, str(corrs.shape[0]), str(steps), str(warmup)], capture_output=True,
                           text=True, timeout=600)
    if r.returncode != 0:
        return {"unavailable": (r.stderr or r.stdout)[-300:]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    return {"value": d["value"], "unit": UNIT, "ms_per_step": d["ms_per_step"],
            "h2d_bytes_per_step": int(corrs.shape[0] * 48), "d2h_bytes_per_step": d2h_bytes,
            "path": "C++ rotavote::estimate_single on a fresh std::vector<Correspondence> (pageable), steady_clock"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2502_06337_b200 import synth
    corrs, _, _ = synth.make_config(WORKLOAD)
    threads = os.cpu_count() or 1
    n_sample = args.ref_sample
    kind, times = reference_cpu(n_sample, args.warmup + args.steps, threads, corrs)
    timed = times[args.warmup:]
    per_solve = statistics.mean(timed)
    value = n_sample / per_solve
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_solve * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
            "config": config_block(n_sample, 1),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                             "kind": "reference" if kind.startswith("ref") else "port",
                             "sample": f"estimate_single on {n_sample} of the 1e6 C3 correspondences, "
                                       f"cfg.threads={threads} (only the vote is threaded in the reference)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_device(args):
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2502_06337_b200 as rv
    from paper_2502_06337_b200 import distributed as rvd
    from paper_2502_06337_b200 import synth

    ctx = rv.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    cfg = rv.EstimatorConfig()
    sharded = world > 1 and args.mode == "sharded"
    c = synth.CONFIGS[WORKLOAD]
    if sharded:  # one C3 problem, correspondences sharded across ranks (strong scaling)
        corrs, rots, _ = synth.make_config(WORKLOAD)
        lo, hi = rvd.shard_bounds(corrs.shape[0], world, rank)
        mine = np.ascontiguousarray(corrs[lo:hi])
    else:  # independent problem per rank (replicas); rank 0 solves the canonical C3 scene
        corrs, rots, _ = synth.make_scene(c.n, c.outlier_frac, c.sigma, seed=c.seed + 1000 * rank)
        mine = corrs
    n_total = corrs.shape[0]
    n_mine = mine.shape[0]
    d_mine = torch.from_numpy(mine).to(f"cuda:{local}")
    host = torch.empty((n_mine, 6), dtype=torch.float64, pin_memory=True)
    host.numpy()[:] = mine
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MiB > L2
    backend = rvd.DeviceBackend(ctx)

    def solve_device():
        if sharded:
            return rvd.sharded_estimate_single(d_mine, n_total, cfg, backend)
        return ctx.estimate_single_device(d_mine.data_ptr(), n_mine, cfg)

    def solve_e2e():
        if sharded:  # H2D of this rank's shard inside the step, then the sharded solve
            d_mine.copy_(host, non_blocking=True)
            return rvd.sharded_estimate_single(d_mine, n_total, cfg, backend)
        return ctx.estimate_single(host.numpy(), cfg)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    warm = max(3, args.warmup)
    for _ in range(warm):
        solve_device()
        solve_e2e()
    # (A) timed device-resident solves (stage timers off: no extra events or read-backs)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            barrier()
            a, b = ev[k]
            a.record(stream)
            est = solve_device()
            b.record(stream)
        barrier()
    dev_ms = [a.elapsed_time(b) for a, b in ev]
    # (B) the same solves again with the per-stage CUDA-event timers on: stage breakdown, the vote
    # kernel's own launch time (roofline) and the launch count; not used for `value`
    ctx.enable_timing(True)
    vote_ms, vote_k_ms, launches, stage = [], [], 0, []
    for k in range(args.steps):
        flush.zero_()
        barrier()
        solve_device()
        st = ctx.stage_times()
        vote_ms.append(st["vote_ms"])
        vote_k_ms.append(st["vote_kernel_ms"])
        launches += st["kernel_launches"]
        stage.append(st)
    barrier()
    ctx.enable_timing(False)
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e2e_wall = []
    d2h_bytes = 0
    barrier()
    for k in range(args.steps):
        flush.zero_()
        barrier()
        a, b = ev2[k]
        t0 = time.perf_counter()
        a.record(stream)
        est_h = solve_e2e()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_wall.append(time.perf_counter() - t0)
        d2h_bytes = est_h.inliers.nbytes + 8 * 16
    barrier()
    e2e_ms = [max(a.elapsed_time(b), 1e3 * w) for (a, b), w in zip(ev2, e2e_wall)]

    t_dev = sum(dev_ms) / 1e3
    t_e2e = sum(e2e_ms) / 1e3
    vals = torch.tensor([t_dev, t_e2e, sum(vote_ms) / 1e3, sum(vote_k_ms) / 1e3], dtype=torch.float64,
                        device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    t_dev, t_e2e, t_vote, t_vote_k = vals.tolist()
    total_corrs = (n_total if sharded else n_total * world) * args.steps
    value = total_corrs / t_dev
    e2e_value = total_corrs / t_e2e
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    err_deg = float(np.degrees(np.arccos(np.clip(0.5 * (np.trace(rots[0].T @ est.rotation) - 1), -1, 1))))
    # roofline of the dominant kernel (vote_banded_kernel): algorithmic sample-votes per launch /
    # its average launch time (CUDA events around the kernel on the solve's stream)
    votes_per_launch = n_mine * cfg.theta_samples
    vote_avg_s = t_vote_k / args.steps
    achieved = votes_per_launch / vote_avg_s
    peak = smem_atomic_peak(local)
    prof = vote_profile()
    roof = {"bound": "smem_atomic", "kernel": "vote_banded_kernel",
            "achieved": achieved / 1e9, "peak": (peak / 1e9) if peak else None, "unit": "Gvotes/s",
            "frac": (achieved / peak) if peak else None,
            "traffic": prof.get("dram_bytes_per_launch") if prof else None,
            "peak_source": "conflict-free u32 smem atomicAdd, measured live (tools/microbench)",
            "work_per_launch": f"{votes_per_launch} sample-votes (N*J of this rank)",
            "kernel_ms_per_solve": 1e3 * vote_avg_s, "kernel_share_of_solve": t_vote_k / t_dev,
            "vote_stage_ms_per_solve": 1e3 * t_vote / args.steps,
            "ncu": prof}
    clocks = clk.summary()
    if prof and prof.get("inst_executed") and clocks.get("sm_mhz"):
        # the vote kernel is issue-bound: warp instructions of one launch (ncu) / its live launch
        # time, against 4 issue slots per SM per clock at the sampled SM clock
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        ach = prof["inst_executed"] / vote_avg_s
        pk = 4.0 * sms * clocks["sm_mhz"] * 1e6
        roof["issue"] = {"bound": "instruction issue", "achieved": ach / 1e9, "peak": pk / 1e9,
                         "unit": "G warp-inst/s", "frac": ach / pk,
                         "inst_per_launch": prof["inst_executed"], "source": "ncu inst_executed x live launch time"}
        if prof.get("lsu_wavefronts"):
            # ... and co-bound by the L1 data pipe: one wavefront (LDS/ATOMS/LDG/LDL phase) per clock
            # per SM; its table reads and bank-conflicted shared atomics per launch (ncu) / live time
            ach = prof["lsu_wavefronts"] / vote_avg_s
            pk = 1.0 * sms * clocks["sm_mhz"] * 1e6
            roof["lsu"] = {"bound": "L1 data-pipe wavefronts", "achieved": ach / 1e9, "peak": pk / 1e9,
                           "unit": "G wavefronts/s", "frac": ach / pk,
                           "wavefronts_per_launch": prof["lsu_wavefronts"],
                           "source": "ncu l1tex__data_pipe_lsu_wavefronts.sum x live launch time"}
    pre_ms = statistics.mean(s["preprocess_ms"] for s in stage)
    hbm = measured_peaks().get("hbm_gbs")
    # in-order preprocess (single solves): 48 B read + 24 B of z written per correspondence
    k1_gbs = (72.0 * n_mine) / (pre_ms * 1e-3) / 1e9 if pre_ms > 0 else None
    cpu = cpu1 = None
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        kind, times = reference_cpu(args.cpu_sample, 3, threads, corrs)
        per = statistics.median(times)
        cpu = {"value": args.cpu_sample / per, "unit": UNIT, "cores": threads,
               "kind": "reference" if kind.startswith("ref") else "port",
               "sample": f"reference estimate_single on the first {args.cpu_sample} C3 correspondences, median of "
                         f"3, cfg.threads={threads}"}
        # the reference default (cfg.threads = 1, estimator.hpp:28): one bounded run
        kind1, times1 = reference_cpu(args.cpu_sample, 1, 1, corrs)
        cpu1 = {"value": args.cpu_sample / times1[0], "unit": UNIT, "cores": 1,
                "kind": "reference" if kind1.startswith("ref") else "port",
                "sample": f"reference estimate_single on the first {args.cpu_sample} C3 correspondences, one run, "
                          f"cfg.threads=1 (the reference default)"}
    e2e_pageable = None
    if world == 1 and not args.no_pageable:
        e2e_pageable = pageable_e2e(corrs, args.steps, warm, int(d2h_bytes))
    extra = {"parallelism": (f"sharded{world} (contiguous shards, NCCL all-reduce of the uint32 grid, "
                             f"all-gather of the input)") if sharded else
             (f"replicas{world}" if world > 1 else "single"),
             "solves_per_step": 1 if sharded else world}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic (seeded BASELINE generator, sigma=0.01)",
            "config": config_block(n_total, world, extra),
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": 1e3 * t_e2e / args.steps,
                    "h2d_bytes_per_step": int(n_total * 48 * (1 if sharded else world)),
                    "d2h_bytes_per_step": int(d2h_bytes * (1 if sharded else world))},
            "roofline": roof,
            "roofline_k1": {"bound": "hbm", "kernel": "preprocess_kernel", "achieved": k1_gbs, "peak": hbm,
                            "unit": "GB/s", "frac": (k1_gbs / hbm) if (hbm and k1_gbs) else None,
                            "traffic": None, "bytes_per_corr": 72},
            "stage_ms": {k: statistics.mean(s[k] for s in stage) for k in
                         ("preprocess_ms", "vote_ms", "peaks_ms", "refine_ms", "angles_ms")},
            "e2e_pageable": e2e_pageable,
            "gpu_launches": launches, "cpu_baseline": cpu, "cpu_baseline_1thread": cpu1, "clocks": clocks,
            "accuracy": {"rot_err_deg_vs_truth": err_deg, "inliers": int(est.inliers.size)}}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=1_000_000)
    ap.add_argument("--ref-sample", type=int, default=1_000_000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="sharded", choices=["sharded", "replicas"],
                    help="N>1: shard one C3 problem across ranks (strong) or one problem per rank (weak)")
    ap.add_argument("--no-pageable", action="store_true")
    args = ap.parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:
        # one process per GPU: re-launch this command under torchrun with --gpus ranks
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")            # communicator lines (nranks) ...
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr: stdout keeps the one JSON line
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        os.execvpe(sys.executable, cmd, env)
    if world_env is not None and int(world_env) != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
