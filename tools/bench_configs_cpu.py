"""BASELINE.json configs C1-C4 on the GPU box's HOST cores with the unmodified
reference (oracle/_ref: proj/core -O3 -fopenmp, all host threads), beside
tools/bench_configs.py's B200 numbers. Build times are wall clock around
EdgeStore::build; walk rates use the reference's own WalkStats (hops /
wall_seconds, generate_walks with its default Coop variant); ingest uses
BatchStats::rebuild_duration. Prints one JSON line per measurement."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from oracle.py import Cfg, COracle, RefOracle, ref_available

assert ref_available(), "oracle/_ref not built"
os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
co = COracle()
R = RefOracle()
only = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C4"]
cpu_model = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "")


def emit(**kw):
    print(json.dumps({**kw, "impl": "reference (oracle/_ref)", "threads": int(os.environ["OMP_NUM_THREADS"]),
                      "cpu_model": cpu_model}), flush=True)


def build(edges, mode):
    t0 = time.perf_counter()
    h = R.build_handle(edges, mode)
    return h, time.perf_counter() - t0


def walks(h, cfg, variant=0):
    _, st = R.generate_on(h, cfg, variant=variant)
    return st["hops"], st["wall_seconds"]


if "C1" in only:
    g = co.gen_uniform(100000, 1000000, 1000000, 1)
    best = None
    for _ in range(3):
        h, s = build(g, 0)
        best = s if best is None else min(best, s)
        if _ < 2:
            R.L.twref_store_free(h)
    emit(config="C1", what="build 1M edges", seconds=best, rate=1e6 / best, unit="edges/s")
    for name, bias in (("uniform", 0), ("linear", 1), ("exp_index", 2), ("exp_weight", 3)):
        cfg = Cfg(walk_length=80, start_mode=1, total_walks=100000, bias=bias, start_bias=bias, seed=7)
        r = min((walks(h, cfg) for _ in range(3)), key=lambda x: x[1])
        emit(config="C1", what=f"100K sampled walks L=80 {name}", seconds=r[1], rate=r[0] / r[1], unit="steps/s")
    R.L.twref_store_free(h)

if "C2" in only:
    g = co.gen_uniform(100000, 1000000, 1000000, 1)
    g = g[np.argsort(g[:, 2], kind="stable")]
    for name, bias in (("exp_weight", 3), ("exp_index", 2)):
        cfg = Cfg(walk_length=80, start_mode=1, total_walks=100000, bias=bias, start_bias=0, seed=7)
        out = R.replay(g, 100000, 333333, 0, cfg)
        ing = sum(b[0]["rebuild_duration"] for b in out)
        ws = sum(b[1]["wall_seconds"] for b in out)
        hops = sum(b[1]["hops"] for b in out)
        emit(config="C2", what=f"{len(out)}-batch replay, window 333333, 100K walks/batch {name}", ingest_s=ing,
             walk_s=ws, rate=hops / (ing + ws), unit="steps/s end to end", walk_rate=hops / ws)

if "C3" in only:
    g = co.gen_hub_skewed(10000000, 100000000, 1)
    h, s = build(g, 0)
    emit(config="C3", what=f"build {len(g)} hub-skewed edges", seconds=s, rate=len(g) / s, unit="edges/s")
    del g
    cfg = Cfg(walk_length=80, start_mode=1, total_walks=10000000, bias=1, start_bias=0, seed=7)
    hops, sec = walks(h, cfg)
    emit(config="C3", what="10M sampled walks L=80 linear (Coop)", seconds=sec, rate=hops / sec, unit="steps/s")
    R.L.twref_store_free(h)

if "C4" in only:
    g = co.gen_uniform(10000000, 100000000, 99999999, 4)
    h, s = build(g, 2)
    emit(config="C4", what="build 100M undirected edges + weights + adjacency", seconds=s, rate=len(g) / s,
         unit="edges/s")
    del g
    cfg = Cfg(walk_length=80, start_mode=1, total_walks=10000000, bias=3, start_bias=0, node2vec=1, p=0.5, q=2.0,
              seed=7)
    hops, sec = walks(h, cfg)
    emit(config="C4", what="10M start-edge walks L=80 temporal node2vec (0.5, 2) exp-weight", seconds=sec,
         rate=hops / sec, unit="steps/s")
    R.L.twref_store_free(h)
