"""Edge TSV reader/writer throughput: the device path (twg_parse_edges_tsv /
twg_format_edges_tsv, host bytes in/out) on a C5-batch-sized file vs the
reference's read_edges_tsv / write_edges_tsv (oracle/_ref, one thread) on a
1/50 sample. usage: python tools/bench_edgeio.py [edges]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_16182_b200 as tw  # noqa: E402
from oracle.py import COracle, RefOracle, ref_available  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
co = COracle()
g = co.gen_stream(10_000_000, 0, n, 5) if hasattr(co, "gen_stream") else co.gen_uniform(10_000_000, n, 10**9, 5)
tw.format_edges_tsv(g[:1000])  # warm up the context
t0 = time.perf_counter()
text = tw.format_edges_tsv(g)
fmt_s = time.perf_counter() - t0
t0 = time.perf_counter()
back = tw.read_edges_tsv(text)
parse_s = time.perf_counter() - t0
assert back.shape == g.shape and (back == g).all()
out = {"edges": n, "text_bytes": len(text), "device_format_s": fmt_s, "device_parse_s": parse_s,
       "device_parse_GBps": len(text) / parse_s / 1e9, "device_parse_edges_per_s": n / parse_s,
       "note": "host bytes in/out (pageable numpy buffers), H2D/D2H included"}
if ref_available():
    ref = RefOracle()
    k = max(n // 50, 1)
    sample = text[: text.index(b"\n", len(text) // 50) + 1] if n >= 50 else text
    t0 = time.perf_counter()
    e, err = ref.read_edges_tsv(sample)
    rs = time.perf_counter() - t0
    out["reference_parse_edges_per_s"] = e.shape[0] / rs
    out["reference_sample_edges"] = int(e.shape[0])
# the device path from pinned host memory (what a streaming reader that
# fills pinned buffers sees): H2D + parse, and the SoA result left in HBM
import ctypes as C  # noqa: E402

import torch  # noqa: E402

pin = torch.empty(len(text), dtype=torch.uint8, pin_memory=True)
pin.numpy()[:] = np.frombuffer(text, np.uint8)
lib = tw._abi.load()
ctx = tw.default_context()
best = None
for _ in range(3):
    h, line = C.c_void_p(), C.c_uint64()
    t0 = time.perf_counter()
    assert lib.twg_parse_edges_tsv(ctx.handle, C.c_void_p(pin.data_ptr()), len(text), C.byref(h), C.byref(line)) == 0
    dt = time.perf_counter() - t0
    lib.twg_edges_destroy(h)
    best = dt if best is None else min(best, dt)
out["pinned_parse_to_hbm_s"] = best
out["pinned_parse_to_hbm_GBps"] = len(text) / best / 1e9
out["pinned_parse_to_hbm_edges_per_s"] = n / best
print(json.dumps(out))
