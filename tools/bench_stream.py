#!/usr/bin/env python
"""C5 streaming benchmark (BASELINE.json configs[4]; streaming.py:126-192).

The C2 DC-SBM graph revealed in 10 stages -- (a) emerging: 10 % of a seeded random
arc permutation per stage, (b) snowball: vertices admitted by BFS from 10 seeded
roots -- each stage rebuilding the CSR on the device and running LOBPCG warm-started
from the previous stage's eigenvectors (zero fill for new vertices) or from a fresh
random block, then QRCP. Per stage: seconds (CUDA-synchronised wall clock around the
public ``partition_stream`` stage, as the reference's StageResult.wall_time) and
iterations-to-tolerance; the tolerance is the 10x rule of the final graph that the
reference itself produced (tests/golden/stream_c5.npz).

    python tools/bench_stream.py [--precision float32] [--reference] > c5.json

``--reference`` also runs the unmodified reference (baseline/_ref) on the same stages
with all host BLAS threads, in the same process, for the per-stage comparison.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def stages_for(mode, spec, edges):
    from paper_1708_07481_b200.dcsbm import emerging_slices, snowball_slices

    if mode == "emerging":
        return [(d, spec.n) for d in emerging_slices(edges, 10, seed=spec.seed)]
    return snowball_slices(edges, spec.n, 10, seed=spec.seed)[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="float32")
    ap.add_argument("--reference", action="store_true")
    ap.add_argument("--repeats", type=int, default=2, help="GPU runs per stream (first = warm-up)")
    a = ap.parse_args()
    import torch

    import paper_1708_07481_b200 as spb
    from paper_1708_07481_b200.dcsbm import CONFIGS, generate_dcsbm
    from paper_1708_07481_b200.streaming import StreamStage, partition_stream

    spec = CONFIGS["c2"]
    edges, truth = generate_dcsbm(spec)
    k = spec.blocks
    with np.load(ROOT / "tests" / "golden" / "stream_c5.npz") as g:
        tol, max_iter = float(g["tol"]), int(g["max_iter"])
        gold = {kk: g[kk] for kk in g.files}
    cfg = spb.SolverConfig(block_size=spb.block_size_for(k), tol=tol, max_iter=max_iter, seed=spec.seed)
    out = {"config": "c5: C2 DC-SBM (n=50000, B=44, 1M arcs) in 10 stages, l=49, "
                     f"tol={tol:.6g} (10x rule of the final graph), max_iter={max_iter}",
           "precision": a.precision, "gpu": torch.cuda.get_device_name(0), "streams": {}}
    for mode in ("emerging", "snowball"):
        st = stages_for(mode, spec, edges)
        stages = [StreamStage(index=i + 1, mode=mode, edge_delta=d, n_after=n) for i, (d, n) in enumerate(st)]
        for init in ("warm", "random"):
            res = None
            for _ in range(max(1, a.repeats)):
                torch.cuda.synchronize()
                res = partition_stream(spb.empty_graph(0), stages, cfg, init_mode=init, k_expected=k,
                                       fix_k=True, precision=a.precision)
            key = f"{mode}_{init}"
            out["streams"][key] = {
                "seconds": [round(r.wall_time, 5) for r in res],
                "iterations": [r.iterations for r in res],
                "total_seconds": round(sum(r.wall_time for r in res), 4),
                "total_iterations": int(sum(r.iterations for r in res)),
                "reference_iterations_1thread_here": gold[f"{key}/iterations"].tolist(),
                "reference_seconds_1thread_build_container": gold[f"{key}/seconds"].round(2).tolist(),
            }
            print(key, out["streams"][key]["iterations"], out["streams"][key]["total_seconds"],
                  file=sys.stderr, flush=True)
    if a.reference:
        from threadpoolctl import threadpool_limits

        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        from specpart import graph as rg
        from specpart import lobpcg as rl
        from specpart import streaming as rstr

        threads = os.cpu_count() or 1
        rcfg = rl.SolverConfig(block_size=spb.block_size_for(k), tol=tol, max_iter=max_iter, seed=spec.seed)
        with threadpool_limits(threads):
            for mode in ("emerging", "snowball"):
                st = stages_for(mode, spec, edges)
                stages = [rstr.StreamStage(index=i + 1, mode=mode, edge_delta=d, n_after=n)
                          for i, (d, n) in enumerate(st)]
                for init in ("warm", "random"):
                    t0 = time.perf_counter()
                    res = rstr.partition_stream(rg.empty_graph(0), stages, rcfg, init_mode=init,
                                                k_expected=k, fix_k=True)
                    key = f"{mode}_{init}"
                    out["streams"][key]["reference_seconds"] = [round(r.wall_time, 3) for r in res]
                    out["streams"][key]["reference_iterations"] = [r.iterations for r in res]
                    out["streams"][key]["reference_total_seconds"] = round(time.perf_counter() - t0, 2)
                    out["streams"][key]["speedup_total"] = round(
                        out["streams"][key]["reference_total_seconds"] / out["streams"][key]["total_seconds"], 1)
                    print(key, "reference", out["streams"][key]["reference_total_seconds"], file=sys.stderr,
                          flush=True)
        out["reference_threads"] = threads
    print(json.dumps(out))


if __name__ == "__main__":
    main()
