#!/usr/bin/env python
"""Full-size oracle parity of the BENCHMARKED path on C4 / C5 by exact cluster
windows (tests/window_check.py explains why the windows are exact), and the
whole-workload CPU oracle timing that falls out of it.

  python tools/window_parity.py --config C4 [--scale 1] [--workers 4]
        [--out profiles/r02/window_parity_C4.json] [--golden tests/golden/window_oracle_C4.json]

1. Build the workload exactly as bench.py does (datagen points, GPU kNN graph,
   eps rule) and run ONE bench step through the C-ABI: kdb_core_mark -> kdb_mst
   -> kdb_label, exact-graph promise, default knobs (filter + fast path on).
2. For every cluster window [s, e): check closure on the device, copy the rows
   to the host with ids shifted by -s, run the CPU oracle (single-threaded,
   ``--workers`` windows at a time, bounded by host RAM), and compare the GPU
   output restricted to the window element by element.
3. The total MSF weight (sum of the windows' oracle weights) against the GPU's
   exactly rounded total within 1e-6 relative.
4. Write the log (per-window times, counts, digests, verdicts) and, with
   --golden, the oracle-only digests keyed by the window's input checksum (the
   cache tests/test_gpu_windows.py checks every window against without
   re-running the oracle).  Stored values come from oracle/ only.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import platform
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (make_workload: the bench's own input recipe)
import paper_2009_04552_b200 as kdb  # noqa: E402
from tests import window_check as wc  # noqa: E402


def gpu_full_run(W):
    N = W["N"]
    g = kdb.Graph(W["nbr"], W["dist"], n_total=N, exact=True)
    ws = torch.empty(kdb.workspace_bytes(g), dtype=torch.uint8, device=W["nbr"].device)
    t = time.perf_counter()
    bits, r, lab = kdb.kdbscan(g, W["M"], W["eps"], workspace=ws)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    full = dict(core=kdb.unpack_core(bits, N).numpy(), comp=r.comp.cpu().numpy(), labels=lab.cpu().numpy(),
                msf_a=r.a.cpu().numpy().astype(np.uint32), msf_b=r.b.cpu().numpy().astype(np.uint32),
                msf_w=r.w.cpu().numpy(), msf_weight=r.weight, count=r.count, stats=r.stats, wall_s=dt)
    del ws
    return full


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4", choices=["C4", "C5"])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--order", default="inertial", choices=["inertial", "generation"],
                    help="point order of the workload (bench.py --order)")
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--windows", default="all", help="'all' or a comma list of window indices")
    ap.add_argument("--out", default=None)
    ap.add_argument("--golden", default=None)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    t0 = time.time()
    W = bench.make_workload(args.config, args.scale, args.seed, torch.device("cuda:0"), order=args.order)
    N, k, M, eps = W["N"], W["k"], W["M"], W["eps"]
    full = gpu_full_run(W)
    wins = wc.cluster_windows(W["truth"])
    sel = range(len(wins)) if args.windows == "all" else [int(x) for x in args.windows.split(",")]
    print(f"[windows] {args.config} x{args.scale}: N={N} k={k} M={M} eps={eps!r} windows={len(wins)} "
          f"gpu step {full['wall_s']:.3f} s", flush=True)
    need = int(36 * k * max(wc.win_size(w) for w in wins) + (1 << 30))
    workers = max(1, min(args.workers, int(wc.MemGate.available() // need), len(sel)))
    log = dict(config=args.config, scale=args.scale, seed=args.seed, order=args.order, N=N, k=k, M=M, eps=eps,
               eps_bits=f"{np.float32(eps).view(np.uint32):08x}", gpu=dict(
                   msf_edges=full["count"], msf_weight=full["msf_weight"], stats=full["stats"]),
               path="kdb_core_mark -> kdb_mst -> kdb_label, KDB_GRAPH_EXACT, default knobs (bench.py step)",
               host=dict(cpu=bench.host_cpu()[0], cores=os.cpu_count(), ram_gb=round(os.sysconf("SC_PAGE_SIZE") *
                                                                                      os.sysconf("SC_PHYS_PAGES") / 2**30, 1),
                         python=platform.python_version()),
               oracle_threads_per_window=1, concurrent_windows=workers, windows=[])
    golden = {}
    results = {}
    t_pool = time.perf_counter()
    def finish(i, win, chk, r):
        got = wc.gpu_window(full, win)
        s, e = win if wc.is_range(win) else (None, None)
        bad = wc.compare(got, r)
        gdig = wc.digest(got["core"], got["labels"], got["msf_a"], got["msf_b"], got["msf_w"])
        results[i] = dict(index=i, s=s, e=e, n=wc.win_size(win), closed=True, input_checksum=chk, ok=not bad,
                          failures=bad,
                          core=int(r["core"].sum()), msf_edges=int(len(r["msf_a"])),
                          oracle_weight=r["msf_weight"], gpu_weight_window=got["msf_weight"],
                          oracle_digest=r["digest"], gpu_digest=gdig,
                          oracle_s=dict(core=r["times"][0], msf=r["times"][1], border=r["times"][2],
                                        wall=r["wall_s"]))
        golden[str(i)] = dict(s=s, e=e, n=wc.win_size(win), input_checksum=chk, oracle_digest=r["digest"],
                              msf_edges=int(len(r["msf_a"])), msf_weight=r["msf_weight"])
        print(f"[window {i}] n={wc.win_size(win)} ok={not bad} {bad} oracle {r['wall_s']:.1f} s "
              f"msf={len(r['msf_a'])}", flush=True)

    with cf.ThreadPoolExecutor(max_workers=workers) as pool:
        running = {}
        for i in sel:
            win = wins[i]
            closed = wc.window_closed(W["nbr"], win)
            chk = wc.input_checksum(W["nbr"], W["dist"], win)
            if not closed:
                results[i] = dict(index=i, n=wc.win_size(win), closed=False, ok=False,
                                  failures=["window not closed"])
                continue
            while len(running) >= workers:  # bound the host copies in flight by the workers
                done, _ = cf.wait(list(running), return_when=cf.FIRST_COMPLETED)
                for f in done:
                    finish(*running.pop(f), f.result())
            nbr_w, dist_w = wc.window_graph_host(W["nbr"], W["dist"], win)
            running[pool.submit(wc.run_oracle, nbr_w, dist_w, M, eps)] = (i, win, chk)
            del nbr_w, dist_w
        for f in cf.as_completed(list(running)):
            finish(*running.pop(f), f.result())
    pool_wall = time.perf_counter() - t_pool
    log["windows"] = [results[i] for i in sorted(results)]
    all_ok = all(w["ok"] for w in log["windows"])
    whole = len(sel) == len(wins)
    if whole:
        tot = float(sum(w["oracle_weight"] for w in log["windows"]))
        cnt = int(sum(w["msf_edges"] for w in log["windows"]))
        log["total"] = dict(oracle_weight_sum=tot, gpu_weight=full["msf_weight"],
                            rel_err=abs(full["msf_weight"] - tot) / tot if tot else 0.0,
                            oracle_msf_edges=cnt, gpu_msf_edges=full["count"])
        all_ok = all_ok and log["total"]["rel_err"] <= 1e-6 and cnt == full["count"]
        one = float(sum(w["oracle_s"]["wall"] for w in log["windows"]))
        log["cpu_baseline_whole_workload"] = dict(
            kind="oracle", unit="edges/s", entries=N * k,
            one_core=dict(seconds=one, value=N * k / one, cores=1,
                          note="sum of the per-window single-threaded oracle runs (the windows are exact, "
                               "independent sub-problems; their sum is the whole workload)"),
            all_cores=dict(seconds=pool_wall, value=N * k / pool_wall, cores=workers,
                           note=f"{len(sel)} windows on {workers} concurrent single-threaded workers "
                                f"(bounded by host RAM: ~36 B per entry per window), wall time incl. D2H"))
    log["ok"] = all_ok
    log["elapsed_s"] = time.time() - t0
    print(json.dumps({k_: v for k_, v in log.items() if k_ != "windows"}, default=str), flush=True)
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        json.dump(log, open(args.out, "w"), indent=1, default=str)
    if args.golden and golden:
        g = dict(config=args.config, scale=args.scale, seed=args.seed, order=args.order, N=N, k=k, M=M,
                 eps_bits=log["eps_bits"],
                 source="tools/window_parity.py: oracle/ (kdb_oracle.cpp) run on each exact cluster window; "
                        "digest = tests/window_check.py digest() of the oracle's window-local outputs",
                 windows=golden)
        if os.path.exists(args.golden):
            old = json.load(open(args.golden))
            if old.get("eps_bits") == g["eps_bits"]:
                old["windows"].update(golden)
                g["windows"] = old["windows"]
        json.dump(g, open(args.golden, "w"), indent=1)
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
