#!/usr/bin/env python3
"""Benchmark of the streaming temporal-walk hot path (BASELINE.json metric:
walk steps/sec + edges ingested/sec over a 1B-edge sliding-window stream).

Workload (BASELINE configs[4]): synthetic power-law stream,
edge i = (src = bits(1,i,0) % N, dst = floor(N*u^3), t = floor(i/4)),
N = 10M nodes, seed 5; batches of 50M edges (batch_duration 12.5M time
units), sliding window Δ = floor(span/3) = 83,333,333 (≈333M-edge window),
ExponentialIndex bias, 10M sampled walks per batch per GPU, L = 80.
One bench "step" = one batch: sliding-window ingest (eviction + full dual
index rebuild on the device) + walk generation on the fresh snapshot.

The window is pre-filled (untimed) to steady state, then W warm-up steps,
then K timed steps (default 7 + 3 + 10 = 20 batches = the 1B-edge stream).

  value      walk steps / s over the timed steps, inputs already in HBM
             (batches pre-generated on the device); edges/s beside it.
  e2e        the same through the reference-facing C ABI with HOST buffers:
             pinned host batch -> twg_window_ingest (H2D inside) ->
             twg_generate -> compact walk download to pinned host memory.
  roofline   walk kernel (k_fullwalk): algorithmic bytes (SURVEY §8d
             B_hop = 80 + 8*ceil(log2(G_v+1)) summed per hop on the device)
             / walk-phase device time, against MEASURED_PEAKS.json hbm_gbs.

Multi-GPU (torchrun): every batch is H2D'd / generated once on rank 0 and
broadcast over NVLink (NCCL) into each rank's replica window; each rank
generates its own 10M walks (disjoint global walk ids) -> weak scaling.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref, unmodified proj/core) on a bounded sample of this workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "walk steps/sec + edges ingested/sec, 1B-edge sliding-window stream, 1–8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="workload scale (1.0 = C5)")
    ap.add_argument("--variant", default="fullwalk", choices=["fullwalk", "coop", "coopdirect"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pipelined", action="store_true",
                    help="headline pass with the walks of batch k overlapping the ingest of k+1 on a second stream "
                         "(measured slower than back to back on B200: both phases compete for HBM)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-audit", action="store_true", help="skip the post-timing causality audit (launch lists)")
    return ap.parse_args()


class Workload:
    def __init__(self, scale: float):
        self.nodes = max(1000, int(10_000_000 * scale))
        self.batch_edges = max(4000, int(50_000_000 * scale))
        self.batch_duration = self.batch_edges // 4          # t = floor(i/4)
        self.total_edges = 20 * self.batch_edges              # 1B at scale 1
        span = self.total_edges // 4
        self.window = span // 3                               # Δ = floor(span/3) (main.cpp:186)
        self.prefill = math.ceil(self.window / self.batch_duration)  # batches to reach steady state
        self.walks = max(1000, int(10_000_000 * scale))
        self.walk_length = 80
        self.seed = 5

    def describe(self, scale):
        return {"workload": "C5: 1B-edge power-law stream, sliding window, exp-index walks"
                if scale == 1.0 else f"C5 shape at scale {scale}",
                "nodes": self.nodes, "batch_edges": self.batch_edges, "window_duration": self.window,
                "window_edges": self.window * 4, "walks_per_batch_per_gpu": self.walks,
                "walk_length": self.walk_length, "bias": "ExponentialIndex", "start": "sampled edges",
                "direction": "DirectedForward", "prefill_batches": self.prefill,
                "l2": "inputs larger than L2 (window ~16 GB at scale 1)"}


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        # nvidia-smi's start-up holds driver locks that stall CUDA API calls:
        # let it initialise (first sample written) before the timed region.
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.first = self.proc.stdout.readline()
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        out = (getattr(self, "first", "") or "") + out
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- ours

def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_16182_b200 as tw

    torch.cuda.set_device(local_rank)
    wl = Workload(args.scale)
    ctx = tw.Context(local_rank, priority=1)  # ingest: the pipeline's critical path
    stream = torch.cuda.ExternalStream(ctx.stream)
    ctx_w = tw.Context(local_rank)  # walk stream: overlaps the next batch's ingest in the pipelined pass
    wstream = torch.cuda.ExternalStream(ctx_w.stream)
    variant = {"fullwalk": tw.Variant.FullWalk, "coop": tw.Variant.Coop, "coopdirect": tw.Variant.CoopDirect}[
        args.variant]
    B = wl.batch_edges

    group = None
    if world > 1:
        # the product's multi-GPU path: a ReplicaGroup (twg_group_*, NCCL over
        # NVLink) — rank 0 creates the rendezvous id, torch.distributed only
        # carries those 128 bytes
        uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local_rank}")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(tw.group_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, src=0)
        group = tw.ReplicaGroup(ctx, world, rank, bytes(uid.cpu().numpy().tobytes()))

    def walk_cfg():
        # weak scaling: every rank generates wl.walks walks; the group splits
        # the global id range [0, world * wl.walks) into contiguous shards
        return tw.WalkConfig(walk_length=wl.walk_length, start_mode=tw.StartMode.Sampled,
                             total_walks=wl.walks * world, bias=tw.BiasKind.ExponentialIndex,
                             start_bias=tw.BiasKind.UniformIndex, seed=wl.seed)

    def generate(snap, stats=None, wctx=None):
        if group is not None:
            return group.generate(snap, walk_cfg(), variant=variant, stats=stats)
        return tw.generate_walks(snap, walk_cfg(), variant=variant, stats=stats, ctx=wctx)

    lib = tw._abi.load()

    def synth(buf, b):
        # batch b of the stream, generated on this device (rank 0 only in multi-GPU)
        rc = lib.twg_synth_stream_device(ctx.handle, wl.nodes, b * B, B, wl.seed, buf[0].data_ptr(),
                                         buf[1].data_ptr(), buf[2].data_ptr())
        assert rc == 0, lib.twg_last_error()

    def ptrs(buf):
        return [x.data_ptr() for x in buf] if rank == 0 else [0, 0, 0]

    def stage(slot, buf):
        # rank 0's batch -> every replica's staging slot (16 B/edge over NVLink, group copy stream)
        group.stage_device(slot, 0, *ptrs(buf), B if rank == 0 else 0)

    def ingest(window, buf, slot=None, stats=False):
        """One batch into this rank's replica: multi-GPU through the group
        (staged slot, or stage + ingest), single GPU straight from the buffer."""
        if group is None:
            return window.ingest_batch_device(buf[0].data_ptr(), buf[1].data_ptr(), buf[2].data_ptr(), B,
                                              stats=stats)
        gs = group.ingest_staged(window, slot) if slot is not None else group.ingest_device(
            window, 0, *ptrs(buf), B if rank == 0 else 0)
        assert gs.replicas_agree, f"replica hash disagreement on rank {rank}"
        return gs.local

    def new_buf():
        return [torch.empty(B, dtype=torch.int64, device=f"cuda:{local_rank}") for _ in range(3)]

    def step(window, buf):
        ingest(window, buf)
        snap = window.snapshot()
        st = tw.WalkStats()
        ws = generate(snap, stats=st)
        return st, ws

    # ---- device-resident pass ------------------------------------------------------
    window = tw.WindowManager(wl.window, tw.DirectionMode.DirectedForward, weights=False, adjacency=False, ctx=ctx)
    buf = new_buf()
    b = 0
    for _ in range(wl.prefill):
        if rank == 0:
            synth(buf, b)
        ingest(window, buf)
        b += 1
    for _ in range(args.warmup):
        if rank == 0:
            synth(buf, b)
        st, ws = step(window, buf)
        del ws
        b += 1
    def timed_pass(pipelined, b):
        """K steps of batches b..b+K-1, inputs pre-generated in HBM, timed with
        device events. Sequential: ingest then walks per batch on one stream.
        Pipelined: the walks of batch k run on a second stream (own context)
        while batch k+1 is ingested; ingest k+2 waits for walks k (the window
        protects only the current and the retired snapshot). Every batch is
        ingested and walked in full either way."""
        bufs = []
        for k in range(args.steps):
            x = new_buf()
            if rank == 0:
                synth(x, b + k)
            bufs.append(x)
        ctx.sync()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = ClockSampler(local_rank)
        clocks.start()
        launches0 = ctx.launches + ctx_w.launches
        hops = alg_bytes = ingest_alg = append_alg = 0
        if not pipelined:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * args.steps + 2)]
            ev[0].record(stream)
            if group is not None:
                stage(0, bufs[0])
            for k in range(args.steps):
                if group is not None and k + 1 < args.steps:
                    stage((k + 1) % 2, bufs[k + 1])  # over NVLink while batch k is ingested and walked
                ev[1 + 3 * k].record(stream)
                bst = ingest(window, bufs[k], slot=k % 2 if group is not None else None, stats=True)
                ev[2 + 3 * k].record(stream)
                snap = window.snapshot()
                st = tw.WalkStats()
                ws = generate(snap, stats=st)
                ev[3 + 3 * k].record(stream)
                hops += st.hops
                alg_bytes += st.alg_bytes
                ingest_alg += batch_alg_bytes(snap.info, bst, B)
                append_alg += append_alg_bytes(snap.info, bst, B)
                del ws, snap
            ev[-1].record(stream)
            ctx.sync()
            torch.cuda.synchronize()
            total_ms = ev[0].elapsed_time(ev[-1])
            ing_ms = [ev[1 + 3 * k].elapsed_time(ev[2 + 3 * k]) for k in range(args.steps)]
            walk_ms_k = [ev[2 + 3 * k].elapsed_time(ev[3 + 3 * k]) for k in range(args.steps)]
        else:
            import queue
            import threading
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            iev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            wev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            ready = queue.Queue()
            done = [threading.Event() for _ in range(args.steps)]
            res = [None] * args.steps
            err = []

            def walker():
                try:
                    for k in range(args.steps):
                        snap, bst = ready.get()
                        wev[k][0].record(wstream)
                        st = tw.WalkStats()
                        ws = generate(snap, stats=st, wctx=ctx_w)
                        wev[k][1].record(wstream)
                        res[k] = (st.hops, st.alg_bytes, batch_alg_bytes(snap.info, bst, B),
                                  append_alg_bytes(snap.info, bst, B))
                        del ws, snap
                        done[k].set()
                except Exception as e:  # surfaced in the main thread
                    err.append(e)
                    for d in done:
                        d.set()

            th = threading.Thread(target=walker, daemon=True)
            ev0.record(stream)
            th.start()
            for k in range(args.steps):
                if k >= 2:
                    done[k - 2].wait()
                iev[k][0].record(stream)
                bst = ingest(window, bufs[k], stats=True)
                iev[k][1].record(stream)
                ready.put((window.snapshot(), bst))
            th.join()
            if err:
                raise err[0]
            stream.wait_event(wev[-1][1])
            ev1.record(stream)
            ctx.sync()
            ctx_w.sync()
            torch.cuda.synchronize()
            total_ms = ev0.elapsed_time(ev1)
            ing_ms = [iev[k][0].elapsed_time(iev[k][1]) for k in range(args.steps)]
            walk_ms_k = [wev[k][0].elapsed_time(wev[k][1]) for k in range(args.steps)]
            for h, a, ia, aa in res:
                hops += h
                alg_bytes += a
                ingest_alg += ia
                append_alg += aa
        launches = ctx.launches + ctx_w.launches - launches0
        clk = clocks.stop()
        if os.environ.get("TWG_BENCH_VERBOSE") == "1":
            for k in range(args.steps):
                print(f"{'pipelined' if pipelined else 'sequential'} step {k}: ingest {ing_ms[k]:7.2f} ms  "
                      f"walk {walk_ms_k[k]:7.2f} ms", file=sys.stderr)
        del bufs
        return dict(total_ms=total_ms, ingest_ms=sum(ing_ms), walk_ms=sum(walk_ms_k), hops=hops,
                    alg_bytes=alg_bytes, ingest_alg=ingest_alg, append_alg=append_alg, launches=launches,
                    clocks=clk)

    # sequential pass: the headline, per-phase times and the rooflines (each
    # kernel alone on the GPU); --pipelined adds an overlapped headline pass
    seq = timed_pass(False, b)
    b += args.steps
    # causality audit (GPU, validity.cpp:108-120 semantics) of one full walk
    # generation on the current snapshot, outside the timed region
    audit = walk_output = None
    if not args.no_audit:
        snap = window.snapshot()
        ws = generate(snap)
        audit, _ = ws.audit(snap)
        walk_output = measure_walk_output(tw, ws, lib)
        del ws, snap
    head = timed_pass(True, b) if args.pipelined else seq
    total_ms, launches, clk = head["total_ms"], head["launches"], head["clocks"]
    hops, alg_bytes, ingest_alg = head["hops"], seq["alg_bytes"], seq["ingest_alg"]
    append_alg = seq["append_alg"]
    ingest_ms, walk_ms = seq["ingest_ms"], seq["walk_ms"]
    seq_total_ms, seq_hops = seq["total_ms"], seq["hops"]
    ctx_w.sync()
    del buf, window  # the e2e pass builds its own window: free this one first
    ctx.sync()
    torch.cuda.empty_cache()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    total_ms = allmax(total_ms)
    ingest_ms = allmax(ingest_ms)
    walk_ms = allmax(walk_ms)
    hops_all = allsum(hops)
    edges_all = B * args.steps  # each batch ingested once (replicated on every GPU)
    result = dict(total_ms=total_ms, ingest_ms=ingest_ms, walk_ms=walk_ms, hops=hops_all, edges=edges_all,
                  launches=launches, clocks=clk, alg_bytes=allsum(alg_bytes), ingest_alg=ingest_alg,
                  append_alg=append_alg,
                  seq_total_ms=allmax(seq_total_ms), seq_hops=allsum(seq_hops), pipelined=bool(args.pipelined),
                  audit=audit, walk_output=walk_output)

    # ---- e2e pass through the C ABI with host buffers -----------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, tw, ctx, wl, rank, world, local_rank, variant, walk_cfg, group, generate)
    return result, e2e, wl


def measure_walk_output(tw, ws, lib):
    """The walk writers (io.cpp:119-135 text, :173-183 binary) on one full
    C5 walk generation: device formatting alone, and formatting + D2H into
    pinned host memory (outside the timed region; wall clock around
    synchronous C-ABI calls)."""
    import ctypes as C

    import torch

    n = C.c_uint64()
    t0 = time.perf_counter()
    assert lib.twg_walkset_text(ws.handle, None, 0, C.byref(n)) == 0
    fmt_s = time.perf_counter() - t0
    text_bytes = n.value
    buf = torch.empty(max(text_bytes, 1), dtype=torch.uint8, pin_memory=True)
    t0 = time.perf_counter()
    assert lib.twg_walkset_text(ws.handle, C.c_void_p(buf.data_ptr()), buf.numel(), C.byref(n)) == 0
    text_s = time.perf_counter() - t0
    assert lib.twg_walkset_binary(ws.handle, None, 0, C.byref(n)) == 0
    bin_bytes = n.value
    del buf
    return {"walks": ws.walk_count, "hops": ws.total_hops, "text_bytes": text_bytes,
            "text_format_ms": fmt_s * 1e3, "text_format_plus_d2h_ms": text_s * 1e3,
            "text_GBps": text_bytes / text_s / 1e9, "binary_bytes": bin_bytes,
            "path": "twg_walkset_text (device formatting, pinned D2H); byte-identical to write_walks_text"}


def run_e2e_pipelined(args, tw, ctx, wl, variant, walk_cfg):
    """Single-GPU e2e through the C ABI with host buffers, as a streaming
    consumer would drive it: batch k+1's H2D (twg_stage_batch, copy stream)
    and batch k-1's compact walk D2H (download stream) overlap batch k's
    ingest + walks. Every step's H2D and D2H happen inside the timed region.
    Host batches are generated before timing into pinned memory (a stream
    arrives already in host RAM; generating 50M edges on the host is slower
    than the GPU step)."""
    import ctypes as C

    import psutil
    import torch

    lib = tw._abi.load()
    B = wl.batch_edges
    window = tw.WindowManager(wl.window, tw.DirectionMode.DirectedForward, weights=False, adjacency=False, ctx=ctx)
    dev = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(3)]
    b = 0
    for _ in range(wl.prefill):  # untimed prefill via the device generator
        lib.twg_synth_stream_device(ctx.handle, wl.nodes, b * B, B, wl.seed, dev[0].data_ptr(), dev[1].data_ptr(),
                                    dev[2].data_ptr())
        window.ingest_batch_device(dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr(), B, stats=False)
        b += 1
    del dev
    n_steps = args.warmup + args.steps
    budget = psutil.virtual_memory().available * 0.5
    n_host = max(2, min(n_steps, int(budget // (B * 24))))
    hosts = [torch.empty((B, 3), dtype=torch.int64, pin_memory=True) for _ in range(n_host)]
    for i, h in enumerate(hosts):  # pre-generated input stream (untimed)
        assert lib.twg_synth_stream_host(wl.nodes, (b + i) * B, B, wl.seed, C.c_void_p(h.data_ptr())) == 0
    regenerated = 0  # host buffers refilled inside the loop (host RAM below the whole run's input)
    cap = wl.walks * 8  # entries; grown if needed
    outs = [[torch.empty(wl.walks + 1, dtype=torch.int64, pin_memory=True),
             torch.empty(cap, dtype=torch.int64, pin_memory=True),
             torch.empty(cap, dtype=torch.int64, pin_memory=True)] for _ in range(2)]
    pending = [None, None]
    hops, d2h = 0, 0
    timed_hops = 0
    t_start = None
    assert lib.twg_stage_batch(ctx.handle, 0, C.c_void_p(hosts[0].data_ptr()), B) == 0
    t_prev = time.perf_counter()
    for k in range(n_steps):
        if k == args.warmup:
            ctx.sync()
            for p in pending:
                if p is not None:
                    lib.twg_walkset_wait(p[0].handle)
            t_start = time.perf_counter()
            timed_hops, d2h = 0, 0
        if k + 1 < n_steps:  # H2D of the next batch overlaps this step
            if k + 1 >= n_host:  # buffer reused: refill it with batch k+1 of the stream (its last H2D has landed:
                # the ingest of step k+1-n_host <= k-1 consumed it), so times keep advancing; counted in the timing
                assert lib.twg_synth_stream_host(wl.nodes, (b + k + 1) * B, B, wl.seed,
                                                 C.c_void_p(hosts[(k + 1) % n_host].data_ptr())) == 0
                regenerated += 1
            assert lib.twg_stage_batch(ctx.handle, (k + 1) % 2, C.c_void_p(hosts[(k + 1) % n_host].data_ptr()), B) == 0
        st = tw._abi.twg_batch_stats()
        rc = lib.twg_window_ingest_staged(window.handle, k % 2, None)
        assert rc == 0, lib.twg_last_error()
        snap = window.snapshot()
        wst = tw.WalkStats()
        ws = tw.generate_walks(snap, walk_cfg(), variant=variant, stats=wst)
        slot = k % 2
        if pending[slot] is not None:  # the download two steps back must finish before its buffers are reused
            lib.twg_walkset_wait(pending[slot][0].handle)
            pending[slot] = None
        total = C.c_uint64()
        off, nodes, times = outs[slot]
        rc = lib.twg_walkset_download_compact_async(ws.handle, C.c_void_p(off.data_ptr()), C.c_void_p(nodes.data_ptr()),
                                                    C.c_void_p(times.data_ptr()), nodes.numel(), C.byref(total))
        assert rc == 0, lib.twg_last_error()
        pending[slot] = (ws, total.value)
        if os.environ.get("TWG_BENCH_VERBOSE") == "1":
            now = time.perf_counter()
            print(f"e2e step {k}: {(now - t_prev) * 1e3:7.2f} ms (host loop)", file=sys.stderr)
            t_prev = now
        timed_hops += wst.hops
        d2h += 8 * (ws.walk_count + 1) + 16 * total.value
        del snap
    for p in pending:
        if p is not None:
            lib.twg_walkset_wait(p[0].handle)
    ctx.sync()
    total_s = time.perf_counter() - t_start
    return dict(total_s=total_s, hops=timed_hops, edges=B * args.steps, h2d=B * 24, d2h=d2h / args.steps,
                pipelined=True, host_batches=n_host, host_batches_regenerated_in_loop=regenerated)


def run_e2e(args, tw, ctx, wl, rank, world, local_rank, variant, walk_cfg, group, generate):
    """e2e through the C ABI with host buffers. N=1: run_e2e_pipelined. N>1:
    the ReplicaGroup path — rank 0 stages each host batch (pinned H2D + pack
    to 16 B/edge, twg_group_stage_host), one NCCL broadcast moves it into
    every replica over NVLink while the previous batch is ingested and
    walked, every rank ingests (twg_group_ingest_staged, replica hashes
    all-reduced) and generates its walk shard (twg_group_generate), then
    downloads its compact walks. Per-rank host timing, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    if world == 1:
        return run_e2e_pipelined(args, tw, ctx, wl, variant, walk_cfg)
    lib = tw._abi.load()
    B = wl.batch_edges
    window = tw.WindowManager(wl.window, tw.DirectionMode.DirectedForward, weights=False, adjacency=False, ctx=ctx)
    dev = [torch.empty(B, dtype=torch.int64, device=f"cuda:{local_rank}") for _ in range(3)]
    b = 0
    for _ in range(wl.prefill):  # untimed prefill via the device generator on rank 0
        if rank == 0:
            lib.twg_synth_stream_device(ctx.handle, wl.nodes, b * B, B, wl.seed, dev[0].data_ptr(),
                                        dev[1].data_ptr(), dev[2].data_ptr())
        ptr = [x.data_ptr() for x in dev] if rank == 0 else [0, 0, 0]
        gs = group.ingest_device(window, 0, *ptr, B if rank == 0 else 0)
        assert gs.replicas_agree
        b += 1
    del dev
    n_steps = args.warmup + args.steps
    hosts = []
    if rank == 0:  # the input stream in pinned host RAM (generated untimed)
        hosts = [torch.empty((B, 3), dtype=torch.int64, pin_memory=True) for _ in range(n_steps)]
        for i, h in enumerate(hosts):
            assert lib.twg_synth_stream_host(wl.nodes, (b + i) * B, B, wl.seed, C.c_void_p(h.data_ptr())) == 0

    def stage(k):
        if rank == 0:
            rc = lib.twg_group_stage_host(group.handle, k % 2, 0, C.c_void_p(hosts[k].data_ptr()), B)
        else:
            rc = lib.twg_group_stage_host(group.handle, k % 2, 0, None, 0)
        assert rc == 0, lib.twg_last_error()

    cap = None
    out_off = out_n = out_t = None
    hops, h2d, d2h = 0, 0, 0
    ctx.sync()
    dist.barrier()
    stage(0)
    t0 = None
    for k in range(n_steps):
        if k == args.warmup:
            ctx.sync()
            dist.barrier()
            t0 = time.perf_counter()
            hops, h2d, d2h = 0, 0, 0
        if k + 1 < n_steps:
            stage(k + 1)
        gs = tw._abi.twg_group_batch_stats()
        rc = lib.twg_group_ingest_staged(group.handle, window.handle, k % 2, C.byref(gs))
        assert rc == 0 and gs.replicas_agree, lib.twg_last_error()
        snap = window.snapshot()
        wst = tw.WalkStats()
        ws = generate(snap, stats=wst)
        total = int(ws.total_hops + 2 * ws.walk_count)  # upper bound of recorded entries
        if cap is None or total > cap:
            cap = int(total * 1.25) + 1
            out_off = torch.empty(ws.walk_count + 1, dtype=torch.int64, pin_memory=True)
            out_n = torch.empty(cap, dtype=torch.int64, pin_memory=True)
            out_t = torch.empty(cap, dtype=torch.int64, pin_memory=True)
        rc = lib.twg_walkset_download_compact(ws.handle, C.c_void_p(out_off.data_ptr()), C.c_void_p(out_n.data_ptr()),
                                              C.c_void_p(out_t.data_ptr()))
        assert rc == 0, lib.twg_last_error()
        entries = int(out_off[ws.walk_count].item())
        hops += wst.hops
        h2d += B * 24 if rank == 0 else 0
        d2h += 8 * (ws.walk_count + 1) + 16 * entries
        del ws, snap
    ctx.sync()
    dt = time.perf_counter() - t0

    def allred(x, op):
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=op)
        return float(t.item())

    total_s = allred(dt, dist.ReduceOp.MAX)
    return dict(total_s=total_s, hops=allred(hops, dist.ReduceOp.SUM), edges=B * args.steps,
                h2d=allred(h2d, dist.ReduceOp.SUM) / args.steps, d2h=allred(d2h, dist.ReduceOp.SUM) / args.steps,
                path="ReplicaGroup: twg_group_stage_host (rank 0 pinned H2D + 16-B pack) -> NCCL broadcast -> "
                     "twg_group_ingest_staged -> twg_group_generate -> twg_walkset_download_compact")

CPU_SCALE = 0.1


def cpu_sample_workload():
    """The C5 workload for the CPU reference at the SURVEY §8(d) fallback
    shape, 1/10 scale: same stream law and window/batch ratios (N=1M nodes,
    5M-edge batches, Δ=span/3 -> ~33M-edge window, 1M walks per batch,
    L=80). The window is filled by one window-sized batch (the reference's
    rebuild is O(window) per batch either way, so the steady state is the
    same); every timed step is one 5M-edge batch + its walks."""
    return Workload(CPU_SCALE)


def run_cpu(steps: int, warmup: int, which: str = "reference"):
    """Time the reference's own CPU implementation (oracle/_ref: the
    unmodified proj/core, -O3 -fopenmp, all host threads) on the sample.
    Per step: WindowManager::ingest_batch + generate_walks (Coop, the
    reference default). Times from the reference's own timers
    (BatchStats::rebuild_duration, WalkStats::wall_seconds)."""
    import ctypes as C

    import numpy as np

    from oracle.py import BatchStatsC, Cfg, COracle, RefOracle, ThresholdsC, WalkStatsC, _p, ref_available

    wl = cpu_sample_workload()
    co = COracle()
    use_ref = which == "reference" and ref_available()
    R = RefOracle() if use_ref else None
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    B = wl.batch_edges
    cfg = Cfg(walk_length=wl.walk_length, start_mode=1, total_walks=wl.walks, bias=2, start_bias=0, seed=wl.seed)
    ingest_s = walk_s = 0.0
    hops = edges = 0
    if use_ref:
        L = R.L
        st = C.c_int()
        w = L.twref_window_create(wl.window, 0, C.byref(st))
        e = co.gen_stream(wl.nodes, 0, wl.prefill * B, wl.seed)  # the window in one batch
        bs = BatchStatsC()
        assert L.twref_window_ingest(w, _p(e), wl.prefill * B, C.byref(bs)) == 0
        del e
        for b in range(wl.prefill, wl.prefill + warmup + steps):
            e = co.gen_stream(wl.nodes, b * B, B, wl.seed)
            bs = BatchStatsC()
            rc = L.twref_window_ingest(w, _p(e), B, C.byref(bs))
            assert rc == 0
            snap = L.twref_window_snapshot(w)
            ws = WalkStatsC()
            status = C.c_int()
            th = ThresholdsC(4, 256, 8192, 512, 4096)
            wh = L.twref_generate(snap, C.byref(cfg.c()), C.byref(th), 0, C.byref(ws), C.byref(status))
            L.twref_walks_free(wh)
            L.twref_store_free(snap)
            if b >= wl.prefill + warmup:
                ingest_s += bs.rebuild_duration
                walk_s += ws.wall_seconds
                hops += ws.hops
                edges += B
        L.twref_window_free(w)
        kind = "reference"
    else:  # C restatement (scalar port)
        st = C.c_int()
        Lc = co.L
        w = Lc.two_window_create(wl.window, 0, C.byref(st))
        e = co.gen_stream(wl.nodes, 0, wl.prefill * B, wl.seed)
        bs = BatchStatsC()
        Lc.two_window_ingest(w, _p(e), wl.prefill * B, C.byref(bs))
        for b in range(wl.prefill, wl.prefill + warmup + steps):
            e = co.gen_stream(wl.nodes, b * B, B, wl.seed)
            bs = BatchStatsC()
            Lc.two_window_ingest(w, _p(e), B, C.byref(bs))
            from oracle.py import two_window, two_walkset
            store = C.cast(w, C.POINTER(two_window)).contents.store
            out = two_walkset()
            ws = WalkStatsC()
            Lc.two_generate(store, C.byref(cfg.c()), None, 2, C.byref(out), C.byref(ws))
            Lc.two_walkset_free(C.byref(out))
            if b >= wl.prefill + warmup:
                ingest_s += bs.rebuild_duration
                walk_s += ws.wall_seconds
                hops += ws.hops
                edges += B
        Lc.two_window_free(w)
        kind = "port"
        cores = 1
    total = ingest_s + walk_s
    cpu_model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu_model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return dict(value=hops / total if total else 0.0, edges_per_s=edges / total if total else 0.0,
                ingest_edges_per_s=edges / ingest_s if ingest_s else 0.0,
                walk_steps_per_s=hops / walk_s if walk_s else 0.0, total_s=total, hops=hops, edges=edges,
                kind=kind, cores=cores, cpu_model=cpu_model,
                sample=f"C5 law at 1/{round(1 / CPU_SCALE)} scale (SURVEY 8d fallback shape): N={wl.nodes} nodes, "
                       f"{B}-edge batches, window {wl.window} time units (~{4 * wl.window} edges, filled by one "
                       f"window-sized batch), {wl.walks} exp-index walks/batch, L=80; {steps} timed batches after "
                       f"{warmup} warm-up; reference timers (BatchStats::rebuild_duration + WalkStats::wall_seconds)")


# --------------------------------------------------------------------------- main

def batch_alg_bytes(info, bst, batch_edges, weights=False, adjacency=False) -> int:
    """SURVEY §8(d) algorithmic bytes of one ingest: 24B (input triples) + 16S
    (survivors read) + 32W (merged window written + read for the node view)
    + 12P + 12Q + 12Z + 16V [+ 8P + 8Z weights] [+ 4P + 4V adjacency]."""
    admitted = batch_edges - bst.dropped_late
    W = int(info.edges)
    S = W - admitted
    P, Q, Z, V = int(info.entries), int(info.node_groups), int(info.ts_groups), int(info.nodes)
    b = 24 * batch_edges + 16 * S + 32 * W + 12 * P + 12 * Q + 12 * Z + 16 * V
    if weights:
        b += 8 * P + 8 * Z
    if adjacency:
        b += 4 * P + 4 * V
    return b


def append_alg_bytes(info, bst, batch_edges) -> int:
    """Algorithmic bytes of one STREAMING-APPEND ingest (csrc/append.cu), the
    design's floor: 24B input triples read + 16A log append + 12Zb new ts
    groups + 28Y new node-view entries and marks (Y = A per side) + 8E
    evicted mark times read (E = evicted edges per side) + 64V node meta
    (old read, new written)."""
    A = batch_edges - bst.dropped_late
    W, Z, V = int(info.edges), int(info.ts_groups), int(info.nodes)
    sides = int(info.entries) // max(W, 1)
    Zb = (Z * A) // max(W, 1)
    return 24 * batch_edges + 16 * A + 12 * Zb + 28 * sides * A + 8 * sides * bst.evicted + 64 * V


def walk_traffic(kernel: str = "k_fullwalk"):
    """DRAM bytes per launch of the walk kernel from the committed ncu --set
    full capture (profiles/walk_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "walk_traffic.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_cpu(args.steps, args.warmup, "reference")
        ms = 1000.0 * r["total_s"] / max(args.steps, 1)
        line = {"metric": METRIC, "value": r["value"], "unit": "walk steps/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "impl": "reference", "edges_per_s": r["edges_per_s"],
                "config": {**cpu_sample_workload().describe(CPU_SCALE), "parallelism": "CPU OpenMP"},
                "cpu_baseline": {"value": r["value"], "unit": "walk steps/s", "cores": r["cores"], "kind": r["kind"],
                                 "sample": r["sample"], "cpu_model": r["cpu_model"]},
                "e2e": {"value": r["value"], "unit": "walk steps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "phases": {"ingest_edges_per_s": r["ingest_edges_per_s"],
                           "walk_steps_per_s": r["walk_steps_per_s"]}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))

    res, e2e, wl = run_ours(args, rank, world, local_rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = run_cpu(1, 0, "reference")  # one 1/10-scale batch + walks: ~10-30 s of host work
        except Exception as ex:  # the baseline is reported, never the product path
            cpu = {"value": None, "kind": "unavailable", "cores": 0, "sample": str(ex)}

    if rank == 0:
        peak, peak_src = peaks()
        total_s = res["total_ms"] / 1000.0
        value = res["hops"] / total_s
        walk_s = res["walk_ms"] / 1000.0
        alg = res["alg_bytes"]
        achieved = alg / walk_s / 1e9 if walk_s and alg else None
        line = {
            "metric": METRIC, "value": value, "unit": "walk steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["total_ms"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "edges_per_s": res["edges"] / total_s,
            "multi_gpu": None if world == 1 else {
                "path": "ReplicaGroup (twg_group_*): NCCL broadcast of each batch at 16 B/edge into every replica "
                        "on a copy stream (batch k+1 overlaps batch k), per-batch replica hash all-reduce, walk ids "
                        "sharded by rank", "replicas_agree_every_batch": True,
                "edges_per_s_note": "each replica ingests every batch: edges/s is per replica (flat with N)"},
            "config": {**wl.describe(args.scale), "variant": args.variant, "parallelism": f"replicas{world}+walk-shards",
                       "global_walks_per_batch": wl.walks * world},
            "pipelined": res["pipelined"],
            "causality_audit": {**res["audit"], "scope": "one full walk generation on the steady-state window, "
                                                         "GPU auditor (twg_walkset_audit, EdgeOracle semantics)"}
                               if res["audit"] else None,
            "walk_output": res.get("walk_output"),
            "phases": {"source": "sequential pass (ingest then walks per batch, one stream, device events)",
                       "ms_per_step": res["seq_total_ms"] / args.steps,
                       "ingest_ms_per_step": res["ingest_ms"] / args.steps,
                       "walk_ms_per_step": res["walk_ms"] / args.steps,
                       "ingest_edges_per_s": res["edges"] / (res["ingest_ms"] / 1000.0),
                       "walk_steps_per_s": res["seq_hops"] / walk_s, "hops_per_step": res["hops"] / args.steps},
            "roofline": {"bound": "hbm", "kernel": "k_fullwalk (one launch per step; CUDA events around twg_generate)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": walk_traffic() if args.scale == 1.0 and args.variant == "fullwalk" else None,
                         "algorithmic_bytes_per_launch": alg / args.steps,
                         "per_unit": "B_hop = 80 + 8*ceil(log2(G_v+1)) per hop + 24 per sampled start, summed on device",
                         "peak_source": peak_src},
            "ingest_roofline": {"bound": "hbm", "scope": "whole ingest phase (twg_window_ingest_device)",
                                "achieved": res["append_alg"] / (res["ingest_ms"] / 1000.0) / 1e9, "peak": peak,
                                "unit": "GB/s",
                                "frac": res["append_alg"] / (res["ingest_ms"] / 1000.0) / 1e9 / peak,
                                "algorithmic_bytes_per_batch": res["append_alg"] / args.steps,
                                "per_unit": "streaming append: 24B + 16A + 12Zb + 28Y + 8E + 64V (DESIGN.md 4)",
                                "rebuild_equivalent": {
                                    "bytes_per_batch": res["ingest_alg"] / args.steps,
                                    "per_unit": "24B + 16S + 32W + 12P + 12Q + 12Z + 16V (SURVEY 8d: the "
                                                "reference's full rebuild, which the append route does not do)",
                                    "GBps": res["ingest_alg"] / (res["ingest_ms"] / 1000.0) / 1e9}},
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
        }
        if e2e:
            line["e2e"] = {"value": e2e["hops"] / e2e["total_s"], "unit": "walk steps/s",
                           "edges_per_s": e2e["edges"] / e2e["total_s"],
                           "h2d_bytes_per_step": int(e2e["h2d"]), "d2h_bytes_per_step": int(e2e["d2h"]),
                           "path": ("twg_stage_batch (pinned H2D, copy stream) -> twg_window_ingest_staged -> "
                                    "twg_generate -> twg_walkset_download_compact_async (pinned D2H, download "
                                    "stream); H2D/D2H of neighbouring batches overlap compute")
                           if e2e.get("pipelined") else e2e.get("path")}
        if cpu:
            line["cpu_baseline"] = {"value": cpu.get("value"), "unit": "walk steps/s", "cores": cpu.get("cores"),
                                    "kind": cpu.get("kind"), "sample": cpu.get("sample"),
                                    "edges_per_s": cpu.get("edges_per_s"), "cpu_model": cpu.get("cpu_model")}
        print(json.dumps(line), flush=True)

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
