#!/usr/bin/env python
"""Benchmark: point-to-plane ICP, source-point-iterations/s (BASELINE.json).

A step is one full registration_icp call — target grid build (A1), source
ordering (A2) and max_iterations Gauss-Newton updates (A3-A8) — on the
config named by --config (default: large16m, the HBM-bound 16M/16M config
BASELINE.json's roofline and scaling targets are quoted on). Inputs are
resident in HBM when the timed region starts; they are 576 MB, larger than
the 126 MB L2, so no explicit flush is needed.

value = n_source * updates / step time (whole job, all ranks).
Multi-GPU: torchrun, one process per GPU; every rank replicates the target
grid and owns a contiguous spatial shard of the source; each pass
all-gathers 29 fp64 partial terms (NCCL) and sums them in rank order.

--impl reference times the CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ICP source-point-iterations/sec"
UNIT = "src-pt-it/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="o3g", choices=["o3g", "reference"])
    ap.add_argument("--config", default="large16m")
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--search", type=int, default=1, help="K3 variant: 0 exact fp64 scan, 1 two-pass warp (default), 2 single-pass prefilter, 3 tile-sorted two-pass, 4 smem-staged tiles")
    ap.add_argument("--coop-min", type=int, default=None, help="override O3G_OPT_COOP_MIN")
    ap.add_argument("--src-order", type=int, default=None, help="override O3G_OPT_SOURCE_ORDER")
    ap.add_argument("--prune-min", type=int, default=None, help="override O3G_OPT_PRUNE_MIN")
    ap.add_argument("--interleave", type=int, default=None, help="override O3G_OPT_INTERLEAVE")
    ap.add_argument("--xsort", type=int, default=None, help="override O3G_OPT_XSORT")
    ap.add_argument("--nbr-mask", type=int, default=None, help="override O3G_OPT_NBR_MASK")
    ap.add_argument("--grid", type=int, default=None, help="override O3G_OPT_GRID (1 dense, 2 hashed)")
    ap.add_argument("--regime", default="init", choices=["init", "converged"],
                    help="start from the config's init T (default) or from T* perturbed by 0.1 deg / 1 cm "
                         "(SURVEY 8(d) 'converged-regime' run)")
    ap.add_argument("--bps", type=int, default=None, help="override O3G_OPT_BLOCKS_PER_SM")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--n", type=int, default=None, help="override point count (testing only)")
    return ap.parse_args()


def load_workload(name, n=None):
    """The named BASELINE config. `fragment` carries per-scale parameters and
    its step runs the whole multi-scale driver (downsampling included)."""
    from synth import make
    kw = {"n": n} if (n is not None and name in ("large16m", "fragment", "tiny")) else {}
    return make(name, **kw)


def oracle_view(w):
    """The single registration the CPU oracle samples (finest scale of a
    multi-scale config)."""
    return w["scales"][-1] if "scales" in w else w


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)      # sampler is live before the timed region starts
        except OSError:
            self.proc = None
        self.first = len(self.rows)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = self.rows[max(0, self.first - 1):]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def cpu_oracle_rate(w, budget_s=12.0, seed=2024):
    """Oracle (single thread, as it stands) on a bounded random sample of the
    source: one correspondence + reduction pass per sampled point at init_T."""
    import oracle
    from synth.rng import Stream
    t0 = time.perf_counter()
    grid = oracle.Grid(w["target"], w["dmax"])
    t_grid = time.perf_counter() - t0
    n = len(w["source"])
    k = min(n, 2000)
    idx = Stream(seed).integers(k, n)
    t0 = time.perf_counter()
    oracle.step(w["init_T"], w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid,
                subset=idx)
    dt = time.perf_counter() - t0
    k2 = int(min(n, max(k, k * budget_s / max(dt, 1e-6))))
    idx = Stream(seed + 1).integers(k2, n)
    t0 = time.perf_counter()
    oracle.step(w["init_T"], w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid,
                subset=idx)
    dt = time.perf_counter() - t0
    return dict(value=k2 / dt, unit=UNIT, cores=1, kind="oracle",
                sample=f"{k2} random source points x 1 pass at the start T against the full "
                       f"{len(w['target'])}-point target (single-threaded C oracle, grid build "
                       f"{t_grid:.1f}s excluded)")


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = oracle_view(load_workload(a.config, a.n))
    import oracle
    oracle.build()
    budget = max(2.0, 150.0 / max(1, a.steps + a.warmup))
    vals = []
    for s in range(a.warmup + a.steps):
        r = cpu_oracle_rate(w, budget_s=budget, seed=3000 + s)
        if s >= a.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    cb = dict(vals[-1], value=v)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": None, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": a.config, "n_source": len(w["source"]),
                      "n_target": len(w["target"]), "dmax": w["dmax"]},
           "cpu_baseline": cb,
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist
    import paper_1801_09847_b200 as o3g

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    w = load_workload(a.config, a.n)
    iters = a.iters if a.iters is not None else w["iters"]
    n, m = len(w["source"]), len(w["target"])
    src = torch.from_numpy(w["source"]).to(dev)
    tgt = torch.from_numpy(w["target"]).to(dev)
    nrm = torch.from_numpy(w["target_normals"]).to(dev)
    T0 = w["init_T"]
    if a.regime == "converged":
        from synth.rng import Stream
        from synth.scenes import rigid, rotation
        rs = Stream(0x5EED)
        T0 = w["T_true"] @ rigid(rotation(rs.unit_vectors(1)[0], np.deg2rad(0.1)),
                                 0.01 * rs.unit_vectors(1)[0])
        w = dict(w, init_T=T0)

    ctx = o3g.Context(local)
    ctx.set_option(o3g.o3g.OPT_SEARCH, a.search)
    if a.coop_min is not None:
        ctx.set_option(6, a.coop_min)
    if a.src_order is not None:
        ctx.set_option(8, a.src_order)
    if a.prune_min is not None:
        ctx.set_option(10, a.prune_min)
    if a.interleave is not None:
        ctx.set_option(11, a.interleave)
    if a.xsort is not None:
        ctx.set_option(12, a.xsort)
    if a.nbr_mask is not None:
        ctx.set_option(5, a.nbr_mask)
    if a.grid is not None:
        ctx.set_option(2, a.grid)
    if a.bps is not None:
        ctx.set_option(4, a.bps)
    if world > 1:
        uid = [o3g.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.dist_init(rank, world, uid[0])

    multiscale = "scales" in w
    if multiscale:
        vox = [sc["meta"]["voxel"] for sc in w["scales"]]
        dms = [sc["dmax"] for sc in w["scales"]]
        its = [sc["iters"] if a.iters is None else a.iters for sc in w["scales"]]

    def step(s_, t_, n_):
        """One full registration; returns the source-point-iterations it did."""
        if multiscale:
            r = ctx.run_multiscale(s_, t_, n_, vox, dms, its, init=T0, relative_fitness=0.0,
                                   relative_rmse=0.0)
            return int(np.sum(r["n_source"] * r["iterations"])), r
        ctx.set_target(t_, n_, w["dmax"])
        ctx.set_source(s_, T0)
        r = ctx.run(T0, iters, 0.0, 0.0)
        return n * r.iterations, r

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(a.warmup):
        units, res = step(src, tgt, nrm)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count()
    # inputs smaller than the 126 MB L2 are flushed (a 256 MB write) before
    # every timed step and only the steps themselves are timed
    in_bytes = 12 * n + 24 * m
    flush = in_bytes < 126 * 2 ** 20
    scratch = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev) if flush else None
    with Clocks(local) as clk:
        if not flush:
            ev0.record()
            for _ in range(a.steps):
                units, res = step(src, tgt, nrm)
            ev1.record()
            barrier()
            ms = ev0.elapsed_time(ev1) / a.steps
        else:
            tot = 0.0
            for _ in range(a.steps):
                scratch.fill_(1)
                ev0.record()
                units, res = step(src, tgt, nrm)
                ev1.record()
                torch.cuda.synchronize()
                tot += ev0.elapsed_time(ev1)
            barrier()
            ms = tot / a.steps
    launches = (ctx.launch_count() - l0) // a.steps * a.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = units / (ms / 1e3)

    # per-pass fitness of one (untimed) registration (SURVEY 8(d) config-5 caveat)
    hist_fit = None
    if not multiscale:
        ctx.set_target(tgt, nrm, w["dmax"])
        ctx.set_source(src, T0)
        hist_fit = [round(float(f), 6) for f in ctx.run(T0, iters, 0.0, 0.0, history=True).hist_fitness]

    # dominant kernel (K3) live duration with CUDA events inside the run graph
    ctx.set_option(o3g.o3g.OPT_TIMING, 1)
    t_loop = []
    k3 = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if multiscale:       # K3 of the finest scale (the last run of the driver)
            e0.record()
            units2, r2 = step(src, tgt, nrm)
            e1.record()
        else:
            ctx.set_target(tgt, nrm, w["dmax"])
            ctx.set_source(src, T0)
            e0.record()
            r2 = ctx.run(T0, iters, 0.0, 0.0)
            e1.record()
            units2 = n * r2.iterations
        torch.cuda.synchronize()
        t_loop.append((e0.elapsed_time(e1), units2))
        k3_ms, k3_n, tail_ms = ctx.last_run_kernel_ms()
        k3.append((k3_ms, k3_n, tail_ms))
    ctx.set_option(o3g.o3g.OPT_TIMING, 0)
    k3_ms, k3_n, tail_ms = min(k3)
    k3_avg = k3_ms / k3_n
    hbm, peak_kind = peaks()
    if multiscale:
        n_k3 = int(r2["n_source"][-1])
        m_k3 = len(w["scales"][-1]["target"])
    else:
        n_k3, m_k3 = n, m
    n_local = (rank + 1) * n_k3 // world - rank * n_k3 // world
    alg_bytes = 12 * n_local + 24 * m_k3 / world
    achieved = alg_bytes / (k3_avg / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k3_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{a.config}@{world}")
    loop_ms, loop_units = min(t_loop)

    # e2e: same metric through the C ABI one-shot call with pinned HOST buffers
    e2e = None
    if not a.no_e2e:
        hs = torch.from_numpy(w["source"]).pin_memory()
        ht = torch.from_numpy(w["target"]).pin_memory()
        hn = torch.from_numpy(w["target_normals"]).pin_memory()

        def e2e_step():
            if world == 1 and not multiscale:
                r = o3g.icp_point_to_plane(hs, ht, hn, w["dmax"], T0, iters, 0.0, 0.0)
                return n * r.iterations
            return step(hs, ht, hn)[0]
        e2e_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            r3 = e2e_step()
        e1.record()
        barrier()
        ems = e0.elapsed_time(e1) / a.steps
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": r3 / (ems / 1e3), "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": 12 * n + 24 * m,
               "d2h_bytes_per_step": 472 + 32 + 8 + 4}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        import oracle
        oracle.build()
        cpu = cpu_oracle_rate(oracle_view(w))

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": a.config, "regime": a.regime, "n_source": n, "n_target": m, "dmax": w["dmax"],
                       "iterations": iters, "src_pt_iterations_per_step": units,
                       "scales": ([{"voxel": v, "dmax": d, "iters": k} for v, d, k in zip(vox, dms, its)]
                                  if multiscale else None),
                       "parallelism": f"source-shard x{world}, target grid replicated",
                       "search": ["exact-fp64", "two-pass fp32-prefilter+exact-fp64", "single-pass fp32-prefilter+exact-fp64", "tile-sorted two-pass fp32-prefilter+exact-fp64", "smem-staged-tile two-pass fp32-prefilter+exact-fp64"][a.search],
                       "l2": (f"inputs {in_bytes / 1e6:.0f} MB < 126 MB L2: 256 MB write flushes L2 before "
                              "each timed step" if flush else
                              f"inputs {in_bytes / 1e6:.0f} MB > 126 MB L2 (no flush needed)")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": ["k3_corr_reduce<exact>", "k3_balanced", "k3_corr_reduce<prefilter>",
                                    "k3_sorted", "k3_tiled"][a.search], "kernel_ms": k3_avg,
                         "alg_bytes_per_launch": alg_bytes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "detail": {"loop_ms": loop_ms, "loop_src_pt_it_per_s": loop_units / (loop_ms / 1e3),
                       "k3_total_ms": k3_ms, "tail_total_ms": tail_ms, "k3_launches": k3_n,
                       "fitness": (float(res["fitness"][-1]) if multiscale else res.fitness),
                       "inlier_rmse": (float(res["inlier_rmse"][-1]) if multiscale else res.inlier_rmse),
                       "grid": ctx.grid_info(),
                       "hist_fitness": hist_fit},
        }
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
