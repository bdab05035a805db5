#!/usr/bin/env python
"""Strong-scaling model of the clustering stage from ONE GPU.

Only one B200 is available to this build, so the P-GPU time is modelled from
bench lines measured on one GPU:
  * the 1-GPU line (T_1, per-kernel table), and
  * `bench.py --sim P` lines: the library's sim communicator runs the P ranks'
    work in sequence on one GPU and reports, per virtual rank, the local-first
    phase time (max and sum over ranks), the global phase split into per-rank
    work (offers + ties) and replicated work, the component counts and the
    bytes every collective would carry.

  T_P = core_mark/P + local_max + transition + [global - global_scan - sim_reductions]
        + global_scan/P + filter/P + heavy_rank/P + [heavy - heavy_rank - heavy_sim_reductions]
        + finalize/P + label/P
        + collectives (bytes at the stated bus bandwidth + a latency per call)

Assumptions (stated in the output): NCCL all-reduce / all-gather bus bandwidth
BUSBW GB/s over NVLink 5 / NVSwitch (ring formula: an all-reduce of S bytes
moves 2 (P-1)/P S per rank, an all-gather (P-1)/P S), LAT us per collective.
Usage: python tools/model_scaling.py sim_1.jsonl sim_2.jsonl sim_4.jsonl sim_8.jsonl
"""
from __future__ import annotations

import json
import sys

BUSBW = 700.0   # GB/s, conservative for 8 x B200 NVSwitch (no NVLS assumed)
LAT = 20e-3     # ms per collective


def load(path):
    return [json.loads(l) for l in open(path) if l.strip().startswith("{")][-1]


def kern(line, name):
    return sum(v["ms_per_step"] for k, v in line["kernels"].items() if name in k)


def model(line1, lineP, P):
    T1 = line1["ms_per_step"]
    mst = lineP["mst"]
    ph = mst["phase_ms"]
    lf = mst.get("local_first")
    cm = kern(lineP, "k_core_mark")
    lab = kern(lineP, "k_label")
    # the sim's min-reductions stand in for all-reduces (modelled from the payload);
    # those of the heavy phase are subtracted there
    minred = kern(lineP, "k_min_into") - ph.get("heavy_simred_ms", 0.0)
    pay = mst["payload_bytes_per_rank"]
    rounds = mst["rounds"]
    heavy_rounds = mst["filter"]["heavy_rounds"]
    ar = lambda b: 2.0 * (P - 1) / P * b / (BUSBW * 1e9) * 1e3   # ms
    ag = lambda b: (P - 1) / P * b / (BUSBW * 1e9) * 1e3
    parts = {"core_mark": cm / P, "label": lab / P, "filter": ph["filter_ms"] / P,
             "finalize": ph["finalize_ms"] / P}
    if "heavy_rank_ms" in ph:  # per-rank survivor work divides by P; the sim's reductions are the all-reduce
        parts["heavy: per-rank offers+ties"] = ph["heavy_rank_ms"] / P
        parts["heavy: replicated"] = max(ph["heavy_ms"] - ph["heavy_rank_ms"] - ph["heavy_simred_ms"], 0.0)
    else:
        parts["heavy (replicated)"] = ph["heavy_ms"]
    if lf:
        glob_rep = max(ph["min_edges_ms"] - lf["global_scan_ms"] - minred, 0.0)
        parts.update({"local phase (max rank)": lf["local_ms_max"],
                      "transition all-gather": ag(lf["transition_bytes"]) + 3 * LAT,
                      "global: per-rank offers+ties": lf["global_scan_ms"] / P,
                      "global: replicated": glob_rep})
        n_coll = 2 * (rounds - lf["local_rounds"]) + 2 * heavy_rounds + 6
    else:  # replicated rounds from singletons: the rows phase's offers divide, the rest stays
        parts.update({"rows phase (sim, all ranks)": ph["init_ms"] + ph["min_edges_ms"] - minred})
        n_coll = 2 * rounds + 2 * heavy_rounds + 6
    parts["all-reduce bytes"] = ar(pay["rows"] + pay["heavy"])
    parts["collective latency"] = n_coll * LAT
    TP = sum(parts.values())
    return TP, T1 / (P * TP), parts


def main(paths):
    lines = [load(p) for p in paths]
    line1 = lines[0]
    print(f"T_1 = {line1['ms_per_step']:.2f} ms (measured, 1 GPU, {line1['config']['workload']})")
    print(f"assumptions: all-reduce/all-gather bus bandwidth {BUSBW:.0f} GB/s, {LAT * 1e3:.0f} us per collective")
    for ln in lines[1:]:
        par = ln["config"]["parallelism"]
        P = int(par.split("sim communicator: ")[1].split()[0]) if "sim communicator" in par else ln["n_gpus"]
        TP, eff, parts = model(line1, ln, P)
        lf = ln["mst"].get("local_first")
        print(f"\nP = {P}: modelled T_P = {TP:.2f} ms, efficiency T_1/(P T_P) = {eff:.2f}")
        if lf:
            print(f"  local phase per rank max {lf['local_ms_max']:.2f} ms (sum {lf['local_ms_sum']:.2f}), "
                  f"global components {lf['global_components']}, parked rows {lf['parked_rows']}, "
                  f"local rounds {lf['local_rounds']}")
        for k, v in parts.items():
            print(f"  {k:32s} {v:7.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1:])
