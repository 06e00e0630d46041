#!/usr/bin/env python
"""HER-AHALS outer iterations/s on BASELINE config 2 (300^3, r=20, FP64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c3|c4|c5|c1] [--algo her|ao] [--no-dimtree]

A "step" is one HER-AHALS outer iteration (N block MTTKRPs + N fused AHALS /
extrapolation / Gram updates + the on-device restart decision) over the full
synthetic instance. By default the block MTTKRPs use the dimension tree
(two full tensor passes per iteration: Y_L shared by blocks 0..h-1, Y_R by
blocks h..N-1, h = N-1 for 3-way and N/2 for 4-way; identical algorithm,
summation order only); --no-dimtree runs N full passes. ``value`` is device-timed (CUDA events on the session
stream, tensor resident in HBM; the 216 MB tensor exceeds the 126 MB L2, so no
flush is needed). ``e2e`` is the same metric through the public C-ABI driver
ntf_her_run with host buffers: upload of the tensor and init, K iterations,
download of factors and trace inside the timed region.

``--impl reference`` times the reference algorithm's CPU implementation on the
same config: the oracle restatement in oracle/ (OpenMP over all host cores),
which is pinned to the reference's own sources built in oracle/_ref
(tests/test_ref_build.py). That build links a minimal Eigen stand-in whose
temporaries make it ~10x slower than the restatement at config scale, so
timing it would understate the reference; kind stays "port".

Multi-GPU (torchrun, one rank per GPU): the tensor is slab-sharded along
mode 1; per-GPU work shrinks with N (strong scaling of one instance).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (shape, rank, sigma, dtype, seed, BASELINE.json index, collinear)
    "c1": ([50, 50, 50], 10, 0.01, "f64", 101, 0, False),
    "c2": ([300, 300, 300], 20, 0.0, "f64", 102, 1, False),
    "c3": ([100, 100, 100, 100], 16, 0.01, "f64", 103, 2, False),
    # ill-conditioned: A_i[:, j] = 0.5 s_i + 0.5 U_i[:, j] (collinear factors,
    # SURVEY.md §8(d) rule; bit-tested in tests/test_host_api.py)
    "c4": ([500, 500, 500], 32, 0.01, "f32", 104, 3, True),
    # 32 GB FP32 tensor: generated with the parallel bit-exact generator (a
    # rank of a sharded run generates only its mode-1 slab)
    "c5": ([2000, 2000, 2000], 64, 0.001, "f32", 105, 4, False),
}
LARGE = {"c5"}  # no CPU-oracle leg (the reference algorithm needs minutes per MTTKRP here)
UNIT = "iters/s"


def metric_name(algo):
    return f"{'HER' if algo == 'her' else 'AO'}-AHALS outer iters/s"


def workload_config(cfg_name, algo):
    """The `config` object both arms print (identical dicts)."""
    shape, r, sigma, dt, seed, idx, collinear = CONFIGS[cfg_name]
    return {"workload": f"BASELINE config {idx + 1}: {'x'.join(map(str, shape))} r={r} {dt} sigma={sigma}"
                        f"{' collinear' if collinear else ''} {'HER' if algo == 'her' else 'AO'}-AHALS",
            "seed": seed}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def tree_split(order):
    """Dimension-tree split h of the runtime (runtime.cpp MttkrpEngine):
    N-1 for 3-way tensors, N/2 from 4-way; NTF_TREE_SPLIT overrides."""
    h = order // 2 if order >= 4 else order - 1
    if os.environ.get("NTF_TREE_SPLIT"):
        h = max(1, min(order - 1, int(os.environ["NTF_TREE_SPLIT"])))
    return h


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, device=0):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower() in ("active", "1")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def make_instance(P, cfg_name, rank_world=(0, 1)):
    """The instance (reference generator semantics); on a sharded run only
    this rank's mode-1 slab is generated (bit-identical to that slice)."""
    shape, rank, sigma, dt, seed, _, collinear = CONFIGS[cfg_name]
    spec = P.SyntheticSpec(shape=shape, rank=rank, noise_sigma=sigma, seed=seed, collinear=collinear)
    r, world = rank_world
    slab = P.slab_range(shape[0], r, world) if world > 1 else None
    t, truth = P.generate(spec, dtype=np.float32 if dt == "f32" else np.float64, slab=slab)
    init = P.random_init(shape, rank, P.stream_seed(seed, 1))
    return t, truth, init


def _oracle_instance(cfg_name):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    shape, rank, sigma, dt, seed, _, collinear = CONFIGS[cfg_name]
    t, truth = O.generate(shape, rank, sigma, False, seed, collinear=collinear)
    if dt == "f32":
        t = t.astype(np.float32)
    init = O.random_init(shape, rank, O.stream_seed(seed, 1))
    return O, t, init


def cpu_reference(cfg_name, algo, steps, warmup, threads=None):
    """The reference algorithm on the host cores (oracle restatement):
    warmup + steps outer iterations, rate over the last `steps`."""
    O, t, init = _oracle_instance(cfg_name)
    if threads:
        O.set_threads(threads)
    iters = warmup + steps
    _, f0, recs = O.run(algo, t, init, max_outer_iters=iters)
    t_start = recs[warmup - 1]["time_s"] if warmup > 0 else 0.0
    dt_steps = recs[-1]["time_s"] - t_start
    return steps / dt_steps, dt_steps


def cpu_sample(cfg_name, algo, budget_s, threads):
    """A bounded sample: outer iterations until `budget_s` of run clock (the
    reference's time budget, checked once per iteration), rate over the
    iterations after the first. Returns (iters/s, iterations timed, seconds)."""
    O, t, init = _oracle_instance(cfg_name)
    prev = O.set_threads(threads)
    try:
        _, _, recs = O.run(algo, t, init, max_time_s=budget_s)
    finally:
        O.set_threads(prev)
    if len(recs) >= 2:
        n, secs = len(recs) - 1, recs[-1]["time_s"] - recs[0]["time_s"]
    else:
        n, secs = 1, recs[0]["time_s"]
    return n / secs, n, secs


def cpu_mttkrp_times(cfg_name, threads, reps=5):
    """Per-mode CPU MTTKRP (the reference's materialised-Khatri-Rao loop,
    kernels.cpp:161-191), best and median seconds of `reps` calls
    (tools/kernel_bench.cpp:24-33 pattern)."""
    O, t, init = _oracle_instance(cfg_name)
    prev = O.set_threads(threads)
    out = []
    try:
        for m in range(t.ndim):
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                O.mttkrp(t, init, m)
                ts.append(time.perf_counter() - t0)
                if ts[0] > 5.0 and len(ts) >= 3:
                    break
            out.append({"mode": m, "best_s": min(ts), "median_s": statistics.median(ts), "calls": len(ts)})
    finally:
        O.set_threads(prev)
    return out


def reference_build_sample(cfg_name, algo, budget_s=4.0):
    """The reference's OWN sources (oracle/_ref/libntf_ref.so, built against
    the Eigen stand-in) on a bounded sample of the same instance: reported
    beside the timed restatement, not instead of it -- the stand-in's
    temporaries make this build several times slower than a real Eigen build
    would be, so it is a lower bound of the reference's speed."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyref
        if not os.path.exists(pyref.LIB_PATH):
            return None
        O, t, init = _oracle_instance(cfg_name)
        _, _, recs = pyref.run(algo, t, init, max_time_s=budget_s)
        if len(recs) >= 2:
            n, secs = len(recs) - 1, recs[-1]["time_s"] - recs[0]["time_s"]
        else:
            n, secs = 1, recs[0]["time_s"]
        return {"value": n / secs, "unit": UNIT, "iterations": n, "seconds": secs,
                "what": "the reference's unmodified sources built against the Eigen stand-in of oracle/ref_build "
                        "(a checker: slower than a real Eigen build; lower bound of the reference's speed)"}
    except Exception as exc:  # the checker is optional here
        return {"unavailable": f"{type(exc).__name__}: {exc}"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    if args.config in LARGE:
        print(json.dumps({"impl": "reference", "unavailable": "the reference algorithm needs the 64 GB FP64 "
                          "tensor and minutes per MTTKRP at this config; its CPU arm runs on c1-c4"}), flush=True)
        return
    rate, secs = cpu_reference(args.config, args.algo, args.steps, args.warmup, threads=cores)
    shape, r, sigma, dt, seed, idx, _ = CONFIGS[args.config]
    ref_build = reference_build_sample(args.config, args.algo)
    line = {
        "impl": "reference", "metric": metric_name(args.algo), "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dt,
        "data": "synthetic (reference generator semantics, seeded)",
        "config": workload_config(args.config, args.algo),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{args.warmup}+{args.steps} outer iterations of the full instance; the "
                                   "oracle restatement of the reference algorithm runs (OpenMP over output "
                                   "rows, materialised Khatri-Rao); it is pinned to the reference's own sources "
                                   "built against an Eigen stand-in (oracle/_ref), which is a checker, not a "
                                   "fair timing target"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if ref_build:
        line["cpu_baseline"]["reference_build"] = ref_build
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2001_04321_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
        uid = [P.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = P.Context(local, rank, world, uid[0])
    else:
        ctx = P.Context(local)

    shape, r, sigma, dt, seed, idx, _ = CONFIGS[args.config]
    t_gen, truth, init = make_instance(P, args.config, (rank, world))
    itemsize = 4 if dt == "f32" else 8
    # the caller's tensor lives in pinned host memory (the e2e contract), so
    # the upload inside the timed e2e region runs at link speed
    pinned = "pinned"
    try:
        buf = torch.empty(t_gen.shape, dtype=torch.float32 if dt == "f32" else torch.float64, pin_memory=True)
        t_local = buf.numpy()
        np.copyto(t_local, t_gen)
        del t_gen
    except Exception as exc:  # pinning refused: pageable memory, said in the line
        t_local, pinned = t_gen, f"pageable ({type(exc).__name__})"
    flags = 0 if args.dimtree else P.RUN_DIRECT  # the dimension tree is the library default
    cfg = P.AoConfig(max_outer_iters=args.warmup + args.steps + 10**6, flags=flags)

    prov = P.GpuDenseProvider(t_local, ctx, full_shape=shape)
    sess = P.Session(prov, init, cfg, P.HerParams(), algo=args.algo)
    stream = torch.cuda.ExternalStream(sess.stream_ptr)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (also builds the CUDA graph)
    sess.step(args.warmup)
    sess.sync()
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sess.step(args.steps)
    e1.record(stream)
    sess.sync()
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = args.steps / (ms / 1e3)

    # kernel-timing pass: CUDA events around every MTTKRP launch (direct launches)
    sess.set_kernel_timing(True)
    sess.step(args.steps)
    sess.sync()
    kms, kcnt, kernels_per_iter = sess.kernel_times()
    sess.set_kernel_timing(False)
    trace = sess.trace()
    n_modes = len(shape)
    per_mode_ms = [kms[i] / max(kcnt[i], 1) for i in range(n_modes)]
    # the roofline kernel is a full MTTKRP pass over the tensor: every mode
    # without the dimension tree; with it the two passes of an iteration,
    # Y_L (timed at block 0) and Y_R (block h; h = N-1 for 3-way: block N-1's
    # own MTTKRP), each timed alone -- the other blocks' per_mode_ms are their
    # tree contractions
    slots = sess.pass_slots()  # which timing slots hold full tensor passes
    avg_ms = sum(per_mode_ms[i] for i in slots) / len(slots)
    local_shape = list(t_local.shape)
    bytes_per = P.mttkrp_bytes(local_shape, r, itemsize)
    flops_per = P.mttkrp_flops(local_shape, r)
    hbm_peak, peak_kind = _peaks()
    achieved_gbs = bytes_per / (avg_ms / 1e3) / 1e9
    traffic = None  # dram bytes per MTTKRP launch from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tb = json.load(fh).get(args.config)
        if tb and world == 1:
            traffic = sum(tb["dram_bytes_per_launch"]) / len(tb["dram_bytes_per_launch"])
    except Exception:
        pass
    sess.close()
    prov.close()  # the device-timed run's tensor goes back to the buffer pool before the e2e runs upload theirs

    # e2e through the public C-ABI driver with host buffers: upload of the
    # tensor (the provider), init, K iterations, factors + trace back to the
    # host; three runs, the median reported (the samples ride along)
    e2e_samples = []
    for _ in range(1 if args.config in LARGE else 3):
        barrier()
        t0 = time.perf_counter()
        prov2 = P.GpuDenseProvider(t_local, ctx, full_shape=shape)
        ecfg = P.AoConfig(max_outer_iters=args.steps, flags=flags)
        if args.algo == "her":
            model, tr2 = P.her_run(prov2, init, ecfg, P.HerParams(), ctx=ctx)
        else:
            model, tr2 = P.ao_run(prov2, init, ecfg, ctx=ctx)
        e2e_s = time.perf_counter() - t0
        prov2.close()
        if world > 1:
            tt = torch.tensor([e2e_s], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        e2e_samples.append(e2e_s)
    e2e_s = statistics.median(e2e_samples)

    line = None
    if rank == 0:
        fp64_peak = 36.8  # measured DFMA TFLOP/s (profiles/fma_peaks_r01.log)
        fp32_peak = 71.7
        cpu = None
        if world == 1 and not args.no_cpu_baseline and args.config not in LARGE:
            cores = os.cpu_count() or 1
            rate, n_it, secs = cpu_sample(args.config, args.algo, args.cpu_budget, cores)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "cpu": cpu_model(),
                   "sample": f"{n_it} outer iterations ({secs:.1f} s) after one warm-up iteration, run under the "
                             f"reference's time budget of {args.cpu_budget:g} s on the full instance (oracle "
                             "restatement of the reference algorithm, OpenMP over all cores)"}
            if args.config != "c4":  # one reference iteration at c4 is minutes on one core
                r1, n1, s1 = cpu_sample(args.config, args.algo, args.cpu_budget, 1)
                cpu["single_thread"] = {"value": r1, "unit": UNIT, "cores": 1, "iterations": n1, "seconds": s1}
            cpu["mttkrp_per_mode"] = cpu_mttkrp_times(args.config, cores)
        line = {
            "metric": metric_name(args.algo), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dt,
            "data": "synthetic (reference generator semantics, seeded; random U[0,1) init)",
            "config": workload_config(args.config, args.algo),
            "run": {"l2": "tensor larger than L2 (no flush)", "parallelism": f"mode-1 slabs x{world}",
                    "dimtree": bool(args.dimtree), "graph": True},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved_gbs / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write per launch)",
                         "kernel": ("MTTKRP full tensor passes of an outer iteration (dimension tree: Y_L at block 0 "
                                    "and the second partial; each timed alone)" if args.dimtree
                                    else "MTTKRP (main kernel, avg over modes)"),
                         "pass_slots": slots,
                         "bytes_per_launch": bytes_per, "avg_launch_ms": avg_ms,
                         "per_mode_ms": per_mode_ms,
                         "fma_tflops": flops_per / (avg_ms / 1e3) / 1e12,
                         "fma_peak_tflops": fp32_peak if dt == "f32" else fp64_peak,
                         "fma_frac": flops_per / (avg_ms / 1e3) / 1e12 / (fp32_peak if dt == "f32" else fp64_peak)},
            "e2e": {"value": args.steps / e2e_s, "unit": UNIT, "samples_s": e2e_samples, "host_memory": pinned,
                    "h2d_bytes_per_step": (t_local.nbytes + init.flat().nbytes) / args.steps,
                    "d2h_bytes_per_step": (init.flat().nbytes + 64 * args.steps) / args.steps},
            "gpu_launches": kernels_per_iter * args.steps,
            "clocks": clocks,
            "final_f": trace.final_f() if trace.records else None,
            "restarts": trace.restart_count(),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    # dimension-tree reuse (NTF_RUN_DIMTREE) is the production path: same
    # algorithm, 2 full tensor passes per outer iteration instead of N
    ap.add_argument("--dimtree", dest="dimtree", action="store_true", default=True)
    ap.add_argument("--no-dimtree", dest="dimtree", action="store_false")
    ap.add_argument("--algo", default="her", choices=["her", "ao"])
    ap.add_argument("--cpu-budget", type=float, default=12.0,
                    help="seconds of reference run clock for each CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
