#!/usr/bin/env python
"""bench.py -- kNN-DBSCAN clustering stage on B200 (BASELINE.json metric:
"kNN-DBSCAN k-NNG edges/sec and % of HBM roofline at 1/2/4/8 B200").

One STEP = one pass of the whole hot path over the
resident k-NN graph of the workload: kdb_core_mark -> kdb_mst -> kdb_label.
value = N*k / (max-over-ranks device time per step)  [edges/s, whole job].

Default workload: BASELINE.json configs[3] (C4: N = 64M points on 10 unit
2-spheres in 3-D, exact kNN graph k = 100, M = 50, eps = 1.5 x median 50th-NN
distance) -- the config the metric's 1/2/4/8-GPU numbers are quoted on.  The
graph (51.2 GB) is built once on the GPU by datagen/ (untimed, reported as
graph_build_s) and is larger than L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kNN-DBSCAN k-NNG edges/sec"
UNIT = "edges/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--scale", type=float, default=1.0, help="shrink every cluster (tests only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--order", default="auto", choices=["auto", "inertial", "generation"],
                    help="point order (= kNN-graph ids): inertial = the paper's inertial partition of the "
                         "data set (PAPER.md:45, datagen/partition.py); generation = the generator's "
                         "cluster-major order; auto = inertial for d <= 5 (C1, C4, C5), generation above "
                         "(PAPER.md:45: the partition 'is effective in lower dimension ... less so in higher')")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--general", action="store_true", help="do not promise an exact graph")
    ap.add_argument("--cpu-sample-rows", type=int, default=1_500_000)
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    ap.add_argument("--edge-cols", default=None,
                    help="candidate edges from the first EDGE_COLS columns ('M' = Def. 6's edge set, "
                         "SURVEY.md 8(f) NEXT 1); default all k (north_star)")
    ap.add_argument("--stage", default="cluster", choices=["cluster", "knng"],
                    help="knng: time the exact kNN-graph builder (SURVEY.md 8(f) NEXT 3) on the points of "
                         "--config instead of the clustering stage; compare with Table 2 (PAPER.md:21-36)")
    ap.add_argument("--sim", type=int, default=0,
                    help="N=1: run the library's sim communicator with this many virtual ranks (every rank's "
                         "work in sequence on one GPU; per-rank local-phase times feed the scaling model, "
                         "DESIGN.md §7)")
    ap.add_argument("--nccl1", action="store_true",
                    help="N=1 through a 1-rank NCCL communicator with every collective issued "
                         "(KDB_NCCL_FORCE=1): the multi-rank host path and its per-round syncs")
    ap.add_argument("--inexact", type=int, default=0,
                    help="also time the paper's inexact MST over P contiguous groups (kdb_mst_inexact, "
                         "SURVEY.md 8(f) NEXT 2) and compare it with the exact step; N=1 only")
    ap.add_argument("--eps-factors", default=None,
                    help="comma list: one step = the whole stage at every eps = f x median D[:, M-1] on "
                         "the same resident graph (Fig. eps_mnist protocol, PAPER.md:459-488)")
    return ap.parse_args()


# --------------------------------------------------------------- helpers ----
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                r = [x.strip() for x in r]
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def median_like_numpy(col):
    """numpy.median of a fp32 column promoted to fp64 (mean of the two middle
    values for even n), on the GPU."""
    import torch
    x = col.double()
    n = x.numel()
    if n % 2:
        return float(torch.kthvalue(x, n // 2 + 1).values)
    a = torch.kthvalue(x, n // 2).values
    b = torch.kthvalue(x, n // 2 + 1).values
    return float((a + b) / 2)


def make_workload(cfg_name: str, scale: float, seed: int, device, rank=0, world=1, order="auto"):
    """Points (numpy, seeded), exact kNN graph on the GPU, eps from the config rule.
    world > 1: this rank's rows [b, e) only (the grid builder searches all points
    for its query rows: knng_grid_rows), so no rank ever holds the whole graph
    (C5: 204.8 GB); eps still comes from the median over ALL rows (the column
    D[:, M-1] is all-gathered)."""
    import torch
    from datagen import CONFIGS, gen_config_points
    from paper_2009_04552_b200.knng import build_knng_brute, build_knng_grid
    cfg = CONFIGS[cfg_name]
    t0 = time.time()
    X, truth = gen_config_points(cfg_name, seed, scale)
    if order == "auto":
        order = "inertial" if X.shape[1] <= 5 else "generation"
    t_part = 0.0
    if order == "inertial":  # the data set is partitioned before clustering
        from datagen.partition import inertial_order
        tp = time.time()
        perm = inertial_order(X, device=device)
        if world > 1:  # every rank must hold the same order: rank 0's permutation, broadcast
            import torch.distributed as tdist
            pt = torch.from_numpy(perm).to(device)
            tdist.broadcast(pt, 0)
            perm = pt.cpu().numpy()
            del pt
        X, truth = X[perm], truth[perm]
        del perm
        t_part = time.time() - tp
    t1 = time.time()
    sliced = False
    if X.shape[1] <= 5:   # uniform-grid cell search (C1, C4, C5)
        if world > 1:
            from paper_2009_04552_b200.dist import rank_rows
            rows = rank_rows(len(X), rank, world)
            nbr, dist, info = build_knng_grid(X, cfg["k"], device=device, rows=rows)
            sliced = True
        else:
            nbr, dist, info = build_knng_grid(X, cfg["k"], device=device)
    else:                 # brute force with exact re-rank (C2 d=50, C3 d=10)
        nbr, dist, info = build_knng_brute(X, cfg["k"], device=device)
    torch.cuda.synchronize()
    t2 = time.time()
    col = dist[:, cfg["M"] - 1].contiguous()
    if sliced:  # the eps rule's median is over every row: gather the column
        from paper_2009_04552_b200.dist import gather_rows
        col = gather_rows(col)
    med = median_like_numpy(col)
    del col
    eps = float(np.float32(cfg["eps_factor"] * med))
    return dict(X=X, truth=truth, nbr=nbr, dist=dist, eps=eps, M=cfg["M"], k=cfg["k"], N=len(X),
                d=X.shape[1], gen_s=t1 - t0, partition_s=t_part, order=order, graph_build_s=t2 - t1, knng=info, med=med, sliced=sliced)


def stage_params(args, W):
    """(edge_cols, [eps ...]) of one step: edge_cols 0 = all k; the eps list is
    the config's eps unless --eps-factors asks for a sweep."""
    ec = 0
    if args.edge_cols:
        ec = W["M"] if args.edge_cols == "M" else int(args.edge_cols)
        if not 1 <= ec <= W["k"]:
            raise SystemExit(f"--edge-cols must be in [1, k={W['k']}] or 'M'")
        ec = 0 if ec == W["k"] else ec
    if args.eps_factors:
        eps_list = [float(np.float32(float(f) * W["med"])) for f in args.eps_factors.split(",")]
    else:
        eps_list = [W["eps"]]
    return ec, eps_list


def stage_desc(ec, eps_list, W):
    d = {}
    if ec:
        d["edge_cols"] = ec
        d["edge_set"] = "first edge_cols columns (Def. 6 direct M-reachability when = M)"
    if len(eps_list) > 1:
        d["eps_sweep"] = eps_list
        d["unit_note"] = "value = N*k*len(eps_sweep) / step time: one step clusters the graph at every eps"
    return d


def workload_desc(cfg_name, W, scale):
    from datagen import CONFIGS
    c = CONFIGS[cfg_name]
    return {"workload": f"{cfg_name} (BASELINE.json configs[{int(cfg_name[1]) - 1}])" +
                        (f" scaled x{scale}" if scale != 1.0 else ""),
            "N": W["N"], "d": W["d"], "k": W["k"], "M": W["M"], "eps": W["eps"],
            "eps_rule": f"fp32({c['eps_factor']} x median D[:, M-1])",
            "graph": "exact kNN, self-excluded, fp32 dist / int32 ids (datagen/csrc/knng.cu " +
                     ("grid builder)" if W["d"] <= 5 else "brute-force builder, fp64 re-rank)"),
            "graph_bytes": int(W["N"]) * int(W["k"]) * 8,
            "order": W["order"] + (" (recursive inertial bisection to 64-point leaves, PAPER.md:45; "
                                   f"{W['partition_s']:.1f} s, untimed input preparation)"
                                   if W["order"] == "inertial" else " (cluster-major, random inside a cluster)"),
            "l2": "no flush: the resident graph (>=1 GB) exceeds the 126 MB L2",
            "graph_build_s": round(W["graph_build_s"], 2)}


def oracle_sample(nbr_rows: np.ndarray, dist_rows: np.ndarray, M: int, eps_list, edge_cols=0):
    """Time the CPU oracle (as it stands) on rows [0, n_s) of the workload at every
    eps of the step; entries pointing at ids >= n_s fall outside the sample and
    are skipped by the oracle."""
    import oracle
    t = time.perf_counter()
    for eps in eps_list:
        r = oracle.kdbscan(nbr_rows, dist_rows, M, np.float32(eps), edge_cols=edge_cols or None)
    dt = time.perf_counter() - t
    return dt, r


# ------------------------------------------------------------ reference ----
def run_reference(args):
    import torch
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the oracle arm
    torch.cuda.set_device(local)
    W = make_workload(args.config, args.scale, args.seed, f"cuda:{local}", order=args.order)
    ec, eps_list = stage_params(args, W)
    ns = min(args.cpu_sample_rows, W["N"])
    nbr = W["nbr"][:ns].cpu().numpy()
    dist = W["dist"][:ns].cpu().numpy()
    del W["nbr"], W["dist"]
    times = []
    for it in range(args.warmup + args.steps):
        dt, _ = oracle_sample(nbr, dist, W["M"], eps_list, ec)
        if it >= args.warmup:
            times.append(dt)
    t = float(np.mean(times))
    value = ns * W["k"] * len(eps_list) / t
    whole = whole_workload_baseline(args.config, args.scale, ec, len(eps_list), W["order"])
    sample = (f"rows [0, {ns}) of {args.config} ({W['order']} order: "
              + ("a compact piece of one cluster" if W["order"] == "inertial" else "cluster-major ids")
              + f"; entries to ids >= {ns} skipped), {ns * W['k']} entries per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(workload_desc(args.config, W, args.scale), **stage_desc(ec, eps_list, W)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu_model": host_cpu()[0], "box_cores": host_cpu()[1],
                             **({"whole_workload_measured": whole} if whole else {})},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, args)


def host_cpu():
    """(model name, logical cores) of the host the oracle baseline runs on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


def dram_budget(args, ec, eps_list):
    """DRAM bytes of one whole step summed over every kernel (ncu, committed:
    profiles/r02/dram_budget_c4.txt, tools/dram_budget.py) against the
    algorithmic bytes -- quoted for the default C4 step, not measured here."""
    if args.config != "C4" or args.scale != 1.0 or ec or len(eps_list) != 1:
        return None
    path = os.path.join(ROOT, "profiles", "r02", "dram_budget_c4.txt")
    if not os.path.exists(path):
        return None
    last = [l for l in open(path) if l.startswith("total")]
    if not last:
        return None
    f = last[-1].split()
    return {"source": os.path.relpath(path, ROOT), "dram_gb_per_step": float(f[2]),
            "algorithmic_gb": round((8.0 * 64e6 * 100 + 4.0 * 64e6 + 64e6 / 8) / 1e9, 2),
            "ratio": float(f[-1])}


def host_ram_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                return round(int(line.split()[1]) / 2**20, 1)
    except OSError:
        pass
    return None


def whole_workload_baseline(cfg_name, scale, ec, n_eps, order="generation"):
    """The oracle on the WHOLE workload, measured once by tools/window_parity.py
    (the ten closed cluster windows of C4 / C5 are exact independent
    sub-problems: the sum of their single-threaded oracle times is the
    whole-workload time) and committed under profiles/r02/ -- quoted, not
    re-run (about 17 min of CPU per config)."""
    if ec or n_eps != 1:
        return None
    tag = {("C4", 1.0): "C4", ("C5", 0.25): "C5q"}.get((cfg_name, scale))
    if tag and order == "inertial":
        tag += "i"
    path = os.path.join(ROOT, "profiles", "r02", f"window_parity_{tag}.json") if tag else None
    if not path or not os.path.exists(path):
        return None
    d = json.load(open(path))
    b = d.get("cpu_baseline_whole_workload")
    if not b:
        return None
    return {"source": os.path.relpath(path, ROOT), "host": d.get("host"),
            "one_core": b["one_core"], "all_cores": b["all_cores"],
            "note": "not re-measured in this run: the committed whole-workload oracle timing of the same "
                    "graph (seed 0), sum over exact cluster windows"}


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")


# ----------------------------------------------------------------- ours ----
def run_ours(args):
    import torch
    import torch.distributed as tdist
    import paper_2009_04552_b200 as kdb

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # tuning options (include/kdb.h kdb_set_option): the KDB_* variables of this
    # process's environment, applied once here -- the library never reads them
    knobs = kdb.options_from_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            tdist.barrier()

    from paper_2009_04552_b200.dist import max_over_ranks, rank_rows
    W = make_workload(args.config, args.scale, args.seed, dev, rank=rank, world=world, order=args.order)
    N, k, M, eps = W["N"], W["k"], W["M"], W["eps"]
    rb, re_ = rank_rows(N, rank, world)
    if world > 1 and not W["sliced"]:  # keep this rank's rows only
        W["nbr"] = W["nbr"][rb:re_].clone()
        W["dist"] = W["dist"][rb:re_].clone()
        torch.cuda.empty_cache()
    comm = kdb.Comm.nccl(rank, world) if world > 1 else None
    if args.nccl1 and world == 1:
        kdb.set_option("KDB_NCCL_FORCE", 1)
        knobs["KDB_NCCL_FORCE"] = 1
        comm = kdb.Comm.nccl_single()
    if args.sim and world == 1:  # P virtual ranks on this GPU (DESIGN.md §7 scaling model)
        comm = kdb.Comm.sim(args.sim)
    ec, eps_list = stage_params(args, W)
    kc = ec or k
    g = kdb.Graph(W["nbr"], W["dist"], n_total=N, row_begin=rb, exact=not args.general, edge_cols=ec)
    ws = torch.empty(kdb.workspace_bytes(g, comm), dtype=torch.uint8, device=dev)
    outs = {"comp": torch.empty(N, dtype=torch.int32, device=dev),
            "a": torch.empty(max(N - 1, 1), dtype=torch.int32, device=dev),
            "b": torch.empty(max(N - 1, 1), dtype=torch.int32, device=dev),
            "w": torch.empty(max(N - 1, 1), dtype=torch.float32, device=dev)}
    lab = torch.empty(max(re_ - rb, 1), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step(graph):
        # an eps sweep reuses the light ELL inside the step (KDB_GRAPH_REUSE:
        # same graph and workspace); the step's first eps always rebuilds it
        for i, e in enumerate(eps_list):
            bits = kdb.core_mark(graph, M, e, comm)
            r = kdb.mst(graph, e, bits, comm, workspace=ws, out=outs, reuse=i > 0)
            lb = kdb.label(graph, e, bits, r.comp, out=lab)
        return bits, r, lb

    for _ in range(args.warmup):
        bits, r, lb = step(g)
    torch.cuda.synchronize()
    # ---- timed region ----------------------------------------------------------
    # `value` comes from K un-instrumented steps; the per-kernel table (and the
    # roofline of the dominant kernel) from K more steps with the library's
    # per-launch CUDA events on (they add host work per launch).
    def timed(instrumented):
        kdb.profile(instrumented)
        kdb.profile_reset()
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st_ = []
        out = None
        for _ in range(args.steps):
            out = step(g)
            st_.append(out[1].stats)  # stats of the step's last eps
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        kdb.profile(False)
        ms_ = e0.elapsed_time(e1) / args.steps
        return max_over_ranks(ms_, dev), st_, out

    clocks = ClockSampler(local)
    kdb.profile_reset()
    ms, stats, (bits, r, lb) = timed(False)
    launches = kdb.launch_count()
    ms_prof, stats_prof, _ = timed(True)
    prof = kdb.profile_read()
    clk = clocks.stop()
    F = len(eps_list)
    value = N * k * F / (ms * 1e-3)
    n_clusters = int(torch.unique(r.comp[r.comp >= 0]).numel()) if rank == 0 else None
    msf_count, msf_weight = r.count, r.weight
    if world > 1:  # multi-rank output: each rank returns the edges of its a-range (kdb.h)
        cnt = torch.tensor([msf_count], dtype=torch.int64, device=dev)
        tdist.all_reduce(cnt)
        msf_count = int(cnt.item())
    # clustering quality against the generator's ground truth (outside the timed
    # region): kdb_nmi on the device
    quality = None
    if world == 1 and W.get("truth") is not None:
        truth = torch.from_numpy(np.ascontiguousarray(W["truth"], np.int32)).to(dev)
        v_nmi, n_cl, n_truth = kdb.nmi(lb[:N].contiguous(), truth)
        quality = {"nmi": v_nmi, "clusters": n_cl, "truth_clusters": n_truth,
                   "convention": "SPEC.md:421-431 (2I/(H(A)+H(B)), noise = one pseudo-cluster)"}
        del truth

    # ---- e2e: host buffers through the public API ---------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, kdb, W, N, k, M, eps_list, ec, rb, re_, comm, ws, outs, dev, world)

    # ---- NEXT 2: the paper's inexact MST against the exact step ---------------------------
    inexact = None
    if args.inexact and world == 1:
        inexact = run_inexact(args, kdb, g, M, eps_list[-1], r, lb, ms, stats[-1], stream, dev)

    # ---- roofline of the dominant kernel ------------------------------------------------
    peaks = measured_peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    kern = {n: v for n, v in prof.items() if not n.startswith("cub")}
    dom = max(kern.items(), key=lambda kv: kv[1][0]) if kern else None
    entries_read = sum(s.get("entries_read", 0) for s in stats) / max(len(stats), 1)
    roof = None
    if dom:
        name, (tot_ms, nl) = dom
        per_launch_ms = tot_ms / nl
        algo_bytes = algo_bytes_per_launch(name, N, kc, world, nl / args.steps, stats)
        achieved = algo_bytes / (per_launch_ms * 1e-3) / 1e9 if algo_bytes else None
        traffic = measured_traffic().get(base_name(name), {}).get("dram_bytes_per_launch")
        roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src, "launches_per_step": nl / args.steps,
                "ms_per_launch": per_launch_ms, "share_of_step": tot_ms / args.steps / ms_prof,
                "instrumented_ms_per_step": ms_prof,
                "algo_bytes_per_launch": algo_bytes}
    t_min_ms = F * (8.0 * N * kc + 4.0 * N + N / 8.0) / (peak * 1e9) * 1e3 / world
    kernels = {}
    for n, v in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        e = {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
        ab = algo_bytes_per_launch(n, N, kc, world, v[1] / args.steps, stats) if v[1] else None
        if ab:
            gbs = ab / (v[0] / v[1] * 1e-3) / 1e9
            e.update(algo_gbs=gbs, frac_of_peak=gbs / peak)
        kernels[n] = e

    # ---- cpu baseline (rank 0, N = 1 only) ------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ns = min(args.cpu_sample_rows, N)
        dt, _ = oracle_sample(W["nbr"][:ns].cpu().numpy(), W["dist"][:ns].cpu().numpy(), M, eps_list, ec)
        cpu = {"value": ns * k * F / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "cpu_model": host_cpu()[0], "box_cores": host_cpu()[1], "host_ram_gb": host_ram_gb(),
               "sample": f"rows [0, {ns}) of the workload ({ns * k} entries; entries to ids >= {ns} skipped), "
                         f"one single-threaded run, {dt:.1f} s"}
        whole = whole_workload_baseline(args.config, args.scale, ec, len(eps_list), W["order"])
        if whole:
            cpu["whole_workload_measured"] = whole

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(workload_desc(args.config, W, args.scale),
                               parallelism=f"row-partitioned x{world}" + (" (1-rank NCCL, collectives forced)"
                                                                           if args.nccl1 and world == 1 else "")
                               + (f" (sim communicator: {args.sim} virtual ranks on one GPU)"
                                  if args.sim and world == 1 else ""),
                               exact_graph=not args.general,
                               knobs=dict(sorted(knobs.items())) or "defaults (no tuning-option overrides)",
                               **stage_desc(ec, eps_list, W)),
                "roofline": roof,
                "stage_roofline": {"t_min_ms": t_min_ms, "frac": t_min_ms / ms,
                                   "bytes": "8 N k + 4 N + N/8 (SURVEY.md 8(d))", "peak": peak},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "quality": quality,
                **({"dram_budget": dram_budget(args, ec, eps_list)} if dram_budget(args, ec, eps_list) else {}),
                **({"inexact": inexact} if inexact else {}),
                "clocks": clk, "kernels": kernels,
                "mst": {"edges": msf_count, "weight": msf_weight, "clusters": n_clusters,
                        "rounds": stats[-1]["rounds"], "stall_rounds": stats[-1]["stall_rounds"],
                        "phase_ms": {k_: stats[-1][k_] for k_ in
                                     ("init_ms", "min_edges_ms", "contract_ms", "filter_ms", "heavy_ms",
                                      "heavy_rank_ms", "heavy_simred_ms",
                                      "finalize_ms")},
                        **({"local_first": stats[-1]["local_first"]} if "local_first" in stats[-1] else {}),
                        "payload_bytes_per_rank": {"rows": stats[-1]["payload_rows_bytes"],
                                                   "heavy": stats[-1]["payload_heavy_bytes"]},
                        "filter": {k_: stats[-1][k_] for k_ in
                                   ("tau", "light_components", "survivors", "heavy_rounds", "fallback",
                                    "filter_exceptions", "filter_slow_entries")}}}
        emit(line, args)
    if comm is not None:
        comm.close()
    if world > 1:
        tdist.destroy_process_group()


KW = 16  # light ELL width (csrc/kdb.cu kW)


def base_name(name):
    """'(k_filter<4, true>)' -> 'k_filter'"""
    return name.strip("()").split("<")[0]


def algo_bytes_per_launch(name, N, k, world, launches_per_step, stats):
    """Algorithmic bytes per launch of kernel `name`: the graph
    bytes the launch must read (8 B per (id, weight) entry, SURVEY.md 8(d);
    4 B per entry where only the id is needed) plus 4 B per vertex for
    vertex-unit kernels.  None for kernels without a graph-byte unit."""
    n_local = N / world
    bn = base_name(name)
    mean = lambda key: float(np.mean([s.get(key, 0) for s in stats])) if stats else 0.0
    if bn == "k_core_mark":
        return 4.0 * n_local + n_local / 8.0            # D[v][M-1] per row + the flag words
    if bn == "k_label":
        return 4.0 * n_local + 4.0 * n_local            # first weight of each row + the label
    if bn == "k_light_ell":
        return n_local * (8.0 * KW + 4.0)               # the first kW entries + D[v][k-1] per row
    if bn == "k_filter":
        return n_local * (4.0 * k + 2.0)                # every id (weights only where needed) + row metadata
    if bn in ("k_light_round", "k_light_quad", "k_light_refill", "k_light_first", "k_offer_round", "k_offer_first"):
        er = mean("entries_read")                       # (J, w) entries scanned, all rounds
        rounds = mean("rounds")
        return 8.0 * er / rounds if er and rounds else None
    if bn == "k_relabel":
        return 8.0 * N                                  # read + write one int32 per vertex
    return None


def measured_traffic():
    """Per-launch DRAM bytes (read + write) per kernel from the committed ncu
    summary (profiles/ncu_traffic.json, written by tools/ncu_traffic.py)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        return {}


def run_inexact(args, kdb, g, M, eps, r_exact, lab_exact, ms_exact, st_exact, stream, dev):
    """Time core_mark -> kdb_mst_inexact(P groups) -> label like the exact step and
    compare: Thm. 3(ii) says the labels agree; the forest weight does not."""
    import torch
    P = int(args.inexact)
    for _ in range(max(args.warmup, 1)):
        bits = kdb.core_mark(g, M, eps)
        ri = kdb.mst_inexact(g, eps, bits, P)
        li = kdb.label(g, eps, bits, ri.comp)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        bits = kdb.core_mark(g, M, eps)
        ri = kdb.mst_inexact(g, eps, bits, P)
        li = kdb.label(g, eps, bits, ri.comp)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_i = e0.elapsed_time(e1) / args.steps
    # the exact step's labels are those of its last eps
    same = bool(torch.equal(li[:g.n_rows], lab_exact[:g.n_rows]))
    return {"groups": P, "ms_per_step": ms_i, "exact_ms_per_step": ms_exact,
            "labels_equal_exact": same, "msf_edges": ri.count, "msf_edges_exact": r_exact.count,
            "msf_weight": ri.weight, "msf_weight_exact": r_exact.weight,
            "weight_ratio": ri.weight / r_exact.weight if r_exact.weight else None,
            "local_components": ri.stats["local_components"], "cut_entries": ri.stats["cut_entries"],
            "allreduce_payload_bytes_per_rank": {
                "exact": st_exact.get("payload_rows_bytes", 0) + st_exact.get("payload_heavy_bytes", 0),
                "inexact": ri.stats["payload_heavy_bytes"],
                "note": "MIN all-reduces over the component arrays (Kc 8 B + Bc 4 B per component and "
                        "round) that P ranks would issue; the inexact local phase needs none"}}


def run_e2e(args, kdb, W, N, k, M, eps_list, ec, rb, re_, comm, ws, outs, dev, world):
    """Same metric through the public API from PINNED HOST buffers: each step copies
    this rank's graph rows host->device and reads the labels back."""
    import torch
    n_rows = re_ - rb
    try:
        h_nbr = torch.empty((n_rows, k), dtype=torch.int32, pin_memory=True)
        h_dist = torch.empty((n_rows, k), dtype=torch.float32, pin_memory=True)
    except Exception as ex:  # pinned allocation failed
        return {"error": f"pinned host allocation failed: {ex}"}
    h_nbr.copy_(W["nbr"])
    h_dist.copy_(W["dist"])
    h_lab = torch.empty(n_rows, dtype=torch.int32, pin_memory=True)
    d_nbr, d_dist = W["nbr"], W["dist"]  # device buffers are overwritten by each step's H2D
    stream = torch.cuda.current_stream()
    steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        d_nbr.copy_(h_nbr, non_blocking=True)
        d_dist.copy_(h_dist, non_blocking=True)
        g = kdb.Graph(d_nbr, d_dist, n_total=N, row_begin=rb, exact=not args.general, edge_cols=ec)
        for i, eps in enumerate(eps_list):
            bits = kdb.core_mark(g, M, eps, comm)
            r = kdb.mst(g, eps, bits, comm, workspace=ws, out=outs, reuse=i > 0)
            lb = kdb.label(g, eps, bits, r.comp)
            h_lab.copy_(lb, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as tdist
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    del h_nbr, h_dist
    return {"value": N * k * len(eps_list) / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": int(n_rows) * k * 8, "d2h_bytes_per_step": int(n_rows) * 4 * len(eps_list)}


# Table 2: GOFMM kNN-graph time, approximate (99% accuracy), on Frontera cores
TABLE2 = {(64_000_000, 3, 100): (1792, 363.0), (64_000_000, 5, 100): (1792, 379.0),
          (64_000_000, 32, 100): (1792, 926.0), (256_000_000, 3, 100): (7168, 583.0),
          (256_000_000, 5, 100): (7168, 628.0)}


def run_knng(args):
    """One step = build the exact kNN graph of the config's points on the GPU
    (grid cell search for d <= 5, certified brute force otherwise); CUDA events
    on the launching stream around the whole call (it synchronises inside)."""
    import torch
    from datagen import CONFIGS, gen_config_points
    from paper_2009_04552_b200.knng import build_knng_brute, build_knng_grid
    rank, world, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    cfg = CONFIGS[args.config]
    X, _ = gen_config_points(args.config, args.seed, args.scale)
    n, d = X.shape
    k = cfg["k"]
    Xd = torch.from_numpy(X).to(dev)
    build = (lambda: build_knng_grid(Xd, k, device=dev)) if d <= 5 else (lambda: build_knng_brute(Xd, k, device=dev))
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        out = build()
        del out
    torch.cuda.synchronize()
    times, info = [], None
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nbr, dist, info = build()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        del nbr, dist
    t = float(np.median(times))
    ref = TABLE2.get((n, d, k))
    line = {"metric": "k-NNG build time", "value": t, "unit": "s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (fp64 re-rank / cell test)", "data": "synthetic",
            "stage": "knng",
            "config": {"workload": f"{args.config} points" + (f" scaled x{args.scale}" if args.scale != 1.0 else ""),
                       "N": n, "d": d, "k": k, "builder": "grid cell search" if d <= 5 else "certified brute force",
                       "exact": True},
            "points_per_s": n / t, "info": info,
            "table2": ({"cores": ref[0], "seconds": ref[1], "accuracy": "99% (GOFMM, approximate)",
                        "note": "another machine and an approximate method: context, not the target"}
                       if ref else None)}
    emit(line, args)


def main():
    args = parse()
    if args.stage == "knng":
        run_knng(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
