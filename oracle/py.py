"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracle.

COracle  -> oracle/_build/libtw_oracle.so       (plain-C restatement)
RefOracle-> oracle/_ref/libtimewalk_ref[_philox].so (the unmodified reference)

Both expose the same small interface so tests can run every check against
either; results are numpy arrays named like the product's store fields.
Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libtw_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtimewalk_ref.so")
REF_PHILOX_SO = os.path.join(HERE, "_ref", "libtimewalk_ref_philox.so")

VP = C.c_void_p
U64 = C.c_uint64
I64 = C.c_int64
I = C.c_int


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a.size else C.c_void_p(0)


def ensure_built() -> None:
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)


class WalkConfigC(C.Structure):
    """== two_walk_config == twref_walk_config (rng in the pad slot)."""
    _fields_ = [("walk_length", C.c_uint32), ("start_mode", C.c_int32), ("walks_per_node", C.c_uint32),
                ("_pad0", C.c_uint32), ("total_walks", U64), ("bias", C.c_int32), ("start_bias", C.c_int32),
                ("node2vec", C.c_int32), ("temporal_adjacency", C.c_int32), ("p", C.c_double), ("q", C.c_double),
                ("direction", C.c_int32), ("rng", C.c_int32), ("seed", U64)]


class ThresholdsC(C.Structure):
    _fields_ = [("w_warp", C.c_uint32), ("block_dim", C.c_uint32), ("w_max", C.c_uint32),
                ("g_warp_cap", C.c_uint32), ("g_block_cap", C.c_uint32)]


class WalkStatsC(C.Structure):
    _fields_ = [("walks", U64), ("hops", U64), ("steps", U64), ("solo", U64), ("warp_cached", U64),
                ("warp_direct", U64), ("block_cached", U64), ("block_direct", U64), ("multi_block", U64),
                ("wall_seconds", C.c_double)]


class BatchStatsC(C.Structure):
    _fields_ = [("ingested", U64), ("dropped_late", U64), ("evicted", U64), ("retained", U64),
                ("rebuild_duration", C.c_double), ("peak_bytes", U64)]


@dataclass
class Cfg:
    """Python-side walk config (mirrors WalkConfig defaults, walk_engine.hpp:36-49)."""
    walk_length: int = 80
    start_mode: int = 0
    walks_per_node: int = 10
    total_walks: int = 0
    bias: int = 3
    start_bias: int = 0
    node2vec: bool = False
    p: float = 1.0
    q: float = 1.0
    temporal_adjacency: bool = False
    direction: int = 0
    seed: int = 0
    rng: int = 0

    def c(self) -> WalkConfigC:
        return WalkConfigC(walk_length=self.walk_length, start_mode=self.start_mode,
                           walks_per_node=self.walks_per_node, total_walks=self.total_walks, bias=self.bias,
                           start_bias=self.start_bias, node2vec=int(self.node2vec),
                           temporal_adjacency=int(self.temporal_adjacency), p=self.p, q=self.q,
                           direction=self.direction, rng=self.rng, seed=self.seed)


def stats_dict(s) -> dict:
    return {k: getattr(s, k) for k, _ in s._fields_}


def edges_array(e) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(e, dtype=np.int64))
    return a.reshape(-1, 3) if a.size else np.zeros((0, 3), np.int64)


# ---------------------------------------------------------------- C oracle

class two_store(C.Structure):
    _fields_ = [("mode", C.c_int), ("m", U64), ("V", U64), ("Z", U64), ("P", U64), ("Q", U64), ("A", U64),
                ("src", VP), ("dst", VP), ("t", VP), ("ext", VP), ("ts_off", VP), ("ts_time", VP), ("ts_w", VP),
                ("n_off", VP), ("n_tsidx", VP), ("mk_time", VP), ("mk_start", VP), ("ref_edge", VP),
                ("wprefix", VP), ("adj_off", VP), ("adj", VP)]


class two_window(C.Structure):
    _fields_ = [("duration", I64), ("mode", C.c_int), ("store", C.POINTER(two_store)), ("t_high", I64),
                ("batch_count", U64)]


class two_walkset(C.Structure):
    _fields_ = [("stride", C.c_uint32), ("walk_count", U64), ("nodes", VP), ("times", VP), ("lengths", VP)]


class ReplayConfigC(C.Structure):
    _fields_ = [("batch_duration", I64), ("window_duration", I64), ("mode", C.c_int32), ("variant", C.c_int32),
                ("generate", C.c_int32), ("keep_walks", C.c_int32), ("walk", WalkConfigC),
                ("thresholds", ThresholdsC)]


class ReplayResultC(C.Structure):
    _fields_ = [("batches", U64), ("ingest", C.POINTER(BatchStatsC)), ("walk", C.POINTER(WalkStatsC)),
                ("walks", C.POINTER(two_walkset))]


def _np(ptr, n, dt):
    if n == 0 or not ptr:
        return np.zeros(0, dt)
    buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dt).copy()


class OracleError(Exception):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code} {msg}")
        self.code = code


class COracle:
    kind = "port"

    def __init__(self):
        ensure_built()
        L = C.CDLL(ORACLE_SO)
        self.L = L
        L.two_build.restype = C.POINTER(two_store)
        L.two_build.argtypes = [VP, U64, I, C.POINTER(I)]
        L.two_store_free.argtypes = [C.POINTER(two_store)]
        for g in ("two_gen_uniform", "two_gen_hub_skewed", "two_gen_time_ladder"):
            getattr(L, g).restype = U64
        L.two_gen_uniform.argtypes = [U64, U64, I64, U64, C.POINTER(VP)]
        L.two_gen_hub_skewed.argtypes = [U64, U64, U64, C.POINTER(VP)]
        L.two_gen_mega_hub.restype = U64
        L.two_gen_mega_hub.argtypes = [C.c_uint32, U64, C.POINTER(VP)]
        L.two_gen_time_ladder.argtypes = [U64, C.c_uint32, U64, C.POINTER(VP)]
        L.two_gen_stream.argtypes = [U64, U64, U64, U64, VP]
        L.two_free.argtypes = [VP]
        L.two_rng_bits.restype = U64
        L.two_rng_bits.argtypes = [I, U64, U64, U64, U64]
        L.two_rng_uniform.restype = C.c_double
        L.two_rng_uniform.argtypes = [I, U64, U64, U64, U64]
        L.two_pick_index.argtypes = [I, C.c_double, U64, C.POINTER(U64)]
        L.two_pick_weighted_range.restype = U64
        L.two_pick_weighted_range.argtypes = [C.c_double, VP, U64, U64, C.c_double]
        L.two_oracle_pick.restype = U64
        L.two_oracle_pick.argtypes = [C.c_double, VP, U64]
        L.two_generate.argtypes = [C.POINTER(two_store), C.POINTER(WalkConfigC), C.POINTER(ThresholdsC), I,
                                   C.POINTER(two_walkset), C.POINTER(WalkStatsC)]
        L.two_walkset_free.argtypes = [C.POINTER(two_walkset)]
        L.two_window_create.restype = VP
        L.two_window_create.argtypes = [I64, I, C.POINTER(I)]
        L.two_window_free.argtypes = [VP]
        L.two_window_ingest.argtypes = [VP, VP, U64, C.POINTER(BatchStatsC)]
        L.two_window_bounds.argtypes = [VP, C.POINTER(I64), C.POINTER(I64)]
        L.two_replay.argtypes = [VP, U64, C.POINTER(ReplayConfigC), C.POINTER(ReplayResultC)]
        L.two_replay_free.argtypes = [C.POINTER(ReplayResultC)]
        L.two_temporal_neighborhood.argtypes = [C.POINTER(two_store), I64, I64, I, C.POINTER(U64)]
        L.two_adjacent.argtypes = [C.POINTER(two_store), C.c_uint32, C.c_uint32]
        L.two_adjacent_after.argtypes = [C.POINTER(two_store), C.c_uint32, C.c_uint32, I64, I]
        L.two_sample_start_edge.restype = U64
        L.two_sample_start_edge.argtypes = [C.POINTER(two_store), I, C.c_double, C.c_double]

    # generators -----------------------------------------------------------
    def _take(self, n, ptr) -> np.ndarray:
        a = _np(ptr.value, 3 * n, np.int64).reshape(-1, 3)
        self.L.two_free(ptr)
        return a

    def gen_uniform(self, nodes, edges, t_max, seed):
        p = VP()
        n = self.L.two_gen_uniform(nodes, edges, t_max, seed, C.byref(p))
        return self._take(n, p)

    def gen_hub_skewed(self, bg_nodes, bg_edges, seed):
        p = VP()
        n = self.L.two_gen_hub_skewed(bg_nodes, bg_edges, seed, C.byref(p))
        return self._take(n, p)

    def gen_mega_hub(self, feeders, seed):
        p = VP()
        n = self.L.two_gen_mega_hub(feeders, seed, C.byref(p))
        return self._take(n, p)

    def gen_time_ladder(self, edges, rungs, seed):
        p = VP()
        n = self.L.two_gen_time_ladder(edges, rungs, seed, C.byref(p))
        return self._take(n, p)

    def gen_stream(self, nodes, first, count, seed):
        out = np.zeros((count, 3), np.int64)
        self.L.two_gen_stream(nodes, first, count, seed, _p(out))
        return out

    def rng_bits(self, kind, seed, walk, hop, ordinal):
        return self.L.two_rng_bits(kind, seed, walk, hop, ordinal)

    def rng_uniform(self, kind, seed, walk, hop, ordinal):
        return self.L.two_rng_uniform(kind, seed, walk, hop, ordinal)

    def pick(self, kind, u, n):
        out = U64()
        rc = self.L.two_pick_index(kind, u, n, C.byref(out))
        if rc:
            raise OracleError(rc)
        return out.value

    def pick_weighted_range(self, u, prefix, begin, end, base):
        pf = np.ascontiguousarray(prefix, dtype=np.float64)
        return self.L.two_pick_weighted_range(u, _p(pf), begin, end, base)

    def oracle_pick(self, u, weights):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        return self.L.two_oracle_pick(u, _p(w), w.size)

    # store ----------------------------------------------------------------------
    def build_handle(self, edges, mode):
        e = edges_array(edges)
        st = I()
        h = self.L.two_build(_p(e), e.shape[0], mode, C.byref(st))
        if not h:
            raise OracleError(st.value)
        return h

    def dump_handle(self, h) -> dict:
        s = h.contents
        d = dict(m=s.m, V=s.V, Z=s.Z, P=s.P, Q=s.Q, A=s.A, mode=s.mode)
        d["src"] = _np(s.src, s.m, np.uint32)
        d["dst"] = _np(s.dst, s.m, np.uint32)
        d["t"] = _np(s.t, s.m, np.int64)
        d["ext"] = _np(s.ext, s.V, np.int64)
        d["src_ext"] = d["ext"][d["src"]] if s.m else np.zeros(0, np.int64)
        d["dst_ext"] = d["ext"][d["dst"]] if s.m else np.zeros(0, np.int64)
        d["ts_off"] = _np(s.ts_off, s.Z + 1, np.uint64)
        d["ts_time"] = _np(s.ts_time, s.Z, np.int64)
        d["ts_w"] = _np(s.ts_w, s.Z, np.float64)
        d["n_off"] = _np(s.n_off, s.V + 1, np.uint64)
        d["n_tsidx"] = _np(s.n_tsidx, s.V + 1, np.uint64)
        d["mk_time"] = _np(s.mk_time, s.Q, np.int64)
        d["mk_start"] = _np(s.mk_start, s.Q, np.uint32)
        d["ref_edge"] = _np(s.ref_edge, s.P, np.uint32)
        d["wprefix"] = _np(s.wprefix, s.P, np.float64)
        d["adj_off"] = _np(s.adj_off, s.V + 1, np.uint64)
        d["adj"] = _np(s.adj, s.A, np.uint32)
        owners = np.repeat(np.arange(s.V, dtype=np.uint32), np.diff(d["n_off"]).astype(np.int64))
        re = d["ref_edge"].astype(np.int64)
        if s.mode == 0:
            d["ref_nbr"] = d["dst"][re]
        elif s.mode == 1:
            d["ref_nbr"] = d["src"][re]
        else:
            d["ref_nbr"] = np.where(d["src"][re] == owners, d["dst"][re], d["src"][re]).astype(np.uint32)
        return d

    def build(self, edges, mode) -> dict:
        h = self.build_handle(edges, mode)
        try:
            return self.dump_handle(h)
        finally:
            self.L.two_store_free(h)

    def generate_on(self, h, cfg: Cfg, thresholds=None, variant=0):
        ws = two_walkset()
        st = WalkStatsC()
        th = ThresholdsC(*(thresholds or (4, 256, 8192, 512, 4096)))
        rc = self.L.two_generate(h, C.byref(cfg.c()), C.byref(th), variant, C.byref(ws), C.byref(st))
        if rc:
            raise OracleError(rc)
        cells = ws.walk_count * ws.stride
        out = dict(stride=ws.stride, walk_count=ws.walk_count, nodes=_np(ws.nodes, cells, np.int64),
                   times=_np(ws.times, cells, np.int64), lengths=_np(ws.lengths, ws.walk_count, np.uint32))
        self.L.two_walkset_free(C.byref(ws))
        return out, stats_dict(st)

    def generate(self, edges, mode, cfg: Cfg, thresholds=None, variant=0):
        h = self.build_handle(edges, mode)
        try:
            return self.generate_on(h, cfg, thresholds, variant)
        finally:
            self.L.two_store_free(h)

    def neighborhood(self, edges, mode, queries, direction):
        h = self.build_handle(edges, mode)
        try:
            out = []
            for v, t in queries:
                o = (U64 * 3)()
                rc = self.L.two_temporal_neighborhood(h, v, t, direction, o)
                if rc:
                    raise OracleError(rc)
                out.append((o[0], o[1], o[2]))
            return out
        finally:
            self.L.two_store_free(h)

    # window ------------------------------------------------------------------------
    def window_run(self, batches, duration, mode, every=False):
        """Ingest batches; returns ([(stats, bounds)], final dump) or, with
        every=True, ([(stats, bounds)], [dump after each batch])."""
        st = I()
        w = self.L.two_window_create(duration, mode, C.byref(st))
        if not w:
            raise OracleError(st.value)
        try:
            stats, dumps = [], []
            for b in batches:
                e = edges_array(b)
                bs = BatchStatsC()
                rc = self.L.two_window_ingest(w, _p(e), e.shape[0], C.byref(bs))
                if rc:
                    raise OracleError(rc)
                lo, hi = I64(), I64()
                rcb = self.L.two_window_bounds(w, C.byref(lo), C.byref(hi))
                stats.append((stats_dict(bs), (lo.value, hi.value) if rcb == 0 else None))
                if every:
                    dumps.append(self.dump_handle(C.cast(w, C.POINTER(two_window)).contents.store))
            if every:
                return stats, dumps
            store = C.cast(w, C.POINTER(two_window)).contents.store
            return stats, self.dump_handle(store)
        finally:
            self.L.two_window_free(w)

    def replay(self, edges, batch_duration, window_duration, mode, cfg: Cfg, thresholds=None, variant=0,
               generate=True):
        e = edges_array(edges)
        rc_cfg = ReplayConfigC(batch_duration=batch_duration, window_duration=window_duration, mode=mode,
                               variant=variant, generate=int(generate), keep_walks=1, walk=cfg.c(),
                               thresholds=ThresholdsC(*(thresholds or (4, 256, 8192, 512, 4096))))
        res = ReplayResultC()
        rc = self.L.two_replay(_p(e), e.shape[0], C.byref(rc_cfg), C.byref(res))
        if rc:
            self.L.two_replay_free(C.byref(res))
            raise OracleError(rc)
        out = []
        for b in range(res.batches):
            ws = res.walks[b]
            cells = ws.walk_count * ws.stride
            walks = dict(stride=ws.stride, walk_count=ws.walk_count, nodes=_np(ws.nodes, cells, np.int64),
                         times=_np(ws.times, cells, np.int64), lengths=_np(ws.lengths, ws.walk_count, np.uint32))
            out.append((stats_dict(res.ingest[b]), stats_dict(res.walk[b]), walks))
        self.L.two_replay_free(C.byref(res))
        return out


# ---------------------------------------------------------------- reference

class ReplayCfgRef(C.Structure):
    _fields_ = [("batch_duration", I64), ("window_duration", I64), ("mode", C.c_int32), ("variant", C.c_int32),
                ("generate", C.c_int32), ("keep_walks", C.c_int32), ("walk", WalkConfigC),
                ("thresholds", ThresholdsC)]


def ref_available(philox: bool = False) -> bool:
    return os.path.exists(REF_PHILOX_SO if philox else REF_SO)


class RefOracle:
    """The unmodified reference core through oracle/ref_shim.cpp."""
    kind = "reference"

    def __init__(self, philox: bool = False):
        path = REF_PHILOX_SO if philox else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        self.philox = philox
        L.twref_last_error.restype = C.c_char_p
        for g in ("twref_gen_uniform", "twref_gen_hub_skewed", "twref_gen_mega_hub", "twref_gen_time_ladder",
                  "twref_store_build", "twref_window_create", "twref_window_snapshot", "twref_generate",
                  "twref_replay", "twref_replay_walks"):
            getattr(L, g).restype = VP
        L.twref_gen_uniform.argtypes = [U64, U64, I64, U64]
        L.twref_gen_hub_skewed.argtypes = [U64, U64, U64]
        L.twref_gen_mega_hub.argtypes = [C.c_uint32, U64]
        L.twref_gen_time_ladder.argtypes = [U64, C.c_uint32, U64]
        L.twref_edges_size.restype = U64
        L.twref_edges_size.argtypes = [VP]
        L.twref_edges_copy.argtypes = [VP, VP]
        L.twref_edges_free.argtypes = [VP]
        L.twref_rng_bits.restype = U64
        L.twref_rng_bits.argtypes = [U64, U64, U64, U64]
        L.twref_rng_uniform.restype = C.c_double
        L.twref_rng_uniform.argtypes = [U64, U64, U64, U64]
        L.twref_pick.argtypes = [I, VP, VP, U64, VP]
        L.twref_pick_weighted_range.argtypes = [C.c_double, VP, U64, U64, U64, C.c_double, C.POINTER(U64)]
        L.twref_oracle_pick.argtypes = [C.c_double, VP, U64, C.POINTER(U64)]
        L.twref_store_build.argtypes = [VP, U64, I, C.POINTER(I)]
        L.twref_store_free.argtypes = [VP]
        L.twref_store_counts.argtypes = [VP, VP]
        L.twref_store_dump.argtypes = [VP, I, VP]
        L.twref_store_adjacent.argtypes = [VP, VP, VP, U64, VP]
        L.twref_store_neighborhood.argtypes = [VP, VP, VP, U64, I, VP]
        L.twref_window_create.argtypes = [I64, I, C.POINTER(I)]
        L.twref_window_free.argtypes = [VP]
        L.twref_window_ingest.argtypes = [VP, VP, U64, C.POINTER(BatchStatsC)]
        L.twref_window_snapshot.argtypes = [VP]
        L.twref_window_bounds.argtypes = [VP, C.POINTER(I64), C.POINTER(I64)]
        L.twref_generate.argtypes = [VP, C.POINTER(WalkConfigC), C.POINTER(ThresholdsC), I,
                                     C.POINTER(WalkStatsC), C.POINTER(I)]
        L.twref_walks_stride.restype = C.c_uint32
        L.twref_walks_stride.argtypes = [VP]
        L.twref_walks_count.restype = U64
        L.twref_walks_count.argtypes = [VP]
        L.twref_walks_copy.argtypes = [VP, VP, VP, VP]
        L.twref_walks_free.argtypes = [VP]
        if hasattr(L, "twref_read_edges_tsv"):
            L.twref_read_edges_tsv.argtypes = [VP, U64, VP, U64, C.POINTER(U64), C.POINTER(U64)]
            L.twref_write_edges_tsv.argtypes = [VP, U64, VP, U64, C.POINTER(U64)]
        if hasattr(L, "twref_walks_serialize"):
            L.twref_walks_serialize.argtypes = [C.c_uint32, U64, VP, VP, VP, I, VP, U64, C.POINTER(U64)]
        L.twref_schedule_step.argtypes = [VP, VP, VP, U64, C.POINTER(ThresholdsC), VP, VP, U64]
        L.twref_replay.argtypes = [VP, U64, C.POINTER(ReplayCfgRef), C.POINTER(U64), C.POINTER(I)]
        L.twref_replay_record.argtypes = [VP, U64, C.POINTER(BatchStatsC), C.POINTER(WalkStatsC)]
        L.twref_replay_walks.argtypes = [VP, U64]
        L.twref_replay_free.argtypes = [VP]
        L.twref_check_walkset.argtypes = [VP, U64, I, C.c_uint32, U64, VP, VP, VP, I, VP]

    def _err(self, rc):
        raise OracleError(rc, (self.L.twref_last_error() or b"").decode())

    def _edges(self, h) -> np.ndarray:
        n = self.L.twref_edges_size(h)
        out = np.zeros((n, 3), np.int64)
        self.L.twref_edges_copy(h, _p(out))
        self.L.twref_edges_free(h)
        return out

    def gen_uniform(self, nodes, edges, t_max, seed):
        return self._edges(self.L.twref_gen_uniform(nodes, edges, t_max, seed))

    def gen_hub_skewed(self, bg_nodes, bg_edges, seed):
        return self._edges(self.L.twref_gen_hub_skewed(bg_nodes, bg_edges, seed))

    def gen_mega_hub(self, feeders, seed):
        return self._edges(self.L.twref_gen_mega_hub(feeders, seed))

    def gen_time_ladder(self, edges, rungs, seed):
        return self._edges(self.L.twref_gen_time_ladder(edges, rungs, seed))

    def rng_bits(self, kind, seed, walk, hop, ordinal):
        return self.L.twref_rng_bits(seed, walk, hop, ordinal)

    def pick_many(self, kind, u, n):
        uu = np.ascontiguousarray(u, dtype=np.float64)
        nn = np.ascontiguousarray(n, dtype=np.uint64)
        out = np.zeros(uu.size, np.uint64)
        rc = self.L.twref_pick(kind, _p(uu), _p(nn), uu.size, _p(out))
        if rc:
            self._err(rc)
        return out

    def pick(self, kind, u, n):
        return int(self.pick_many(kind, [u], [n])[0])

    def build_handle(self, edges, mode):
        e = edges_array(edges)
        st = I()
        h = self.L.twref_store_build(_p(e), e.shape[0], mode, C.byref(st))
        if not h:
            self._err(st.value)
        return h

    def dump_handle(self, h, keys=None) -> dict:
        cnt = np.zeros(8, np.uint64)
        self.L.twref_store_counts(h, _p(cnt))
        m, V, Z, P, Q = (int(x) for x in cnt[:5])
        d = dict(m=m, V=V, Z=Z, P=P, Q=Q, mode=int(cnt[5]), memory_bytes=int(cnt[6]))
        spec = [("src_ext", 0, np.int64, m), ("dst_ext", 1, np.int64, m), ("t", 2, np.int64, m),
                ("src", 3, np.uint32, m), ("dst", 4, np.uint32, m), ("ts_off", 5, np.uint64, Z + 1),
                ("ts_time", 6, np.int64, Z), ("ts_w", 7, np.float64, Z), ("n_off", 8, np.uint64, V + 1),
                ("n_tsidx", 9, np.uint64, V + 1), ("mk_time", 10, np.int64, Q), ("mk_start", 11, np.uint32, Q),
                ("ref_edge", 12, np.uint32, P), ("wprefix", 13, np.float64, P), ("ext", 14, np.int64, V),
                ("ref_nbr", 15, np.uint32, P)]
        for name, fid, dt, n in spec:
            if keys is not None and name not in keys:
                continue
            out = np.zeros(max(n, 1), dt)
            rc = self.L.twref_store_dump(h, fid, _p(out))
            if rc:
                self._err(rc)
            d[name] = out[:n]
        return d

    def build(self, edges, mode) -> dict:
        h = self.build_handle(edges, mode)
        try:
            return self.dump_handle(h)
        finally:
            self.L.twref_store_free(h)

    def adjacent(self, h, a, b) -> np.ndarray:
        aa = np.ascontiguousarray(a, dtype=np.uint32)
        bb = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.zeros(aa.size, np.uint8)
        self.L.twref_store_adjacent(h, _p(aa), _p(bb), aa.size, _p(out))
        return out.astype(bool)

    def generate_on(self, h, cfg: Cfg, thresholds=None, variant=0):
        st = WalkStatsC()
        status = I()
        th = ThresholdsC(*(thresholds or (4, 256, 8192, 512, 4096)))
        w = self.L.twref_generate(h, C.byref(cfg.c()), C.byref(th), variant, C.byref(st), C.byref(status))
        if not w:
            self._err(status.value)
        stride = self.L.twref_walks_stride(w)
        count = self.L.twref_walks_count(w)
        nodes = np.zeros(count * stride, np.int64)
        times = np.zeros(count * stride, np.int64)
        lengths = np.zeros(count, np.uint32)
        self.L.twref_walks_copy(w, _p(nodes), _p(times), _p(lengths))
        self.L.twref_walks_free(w)
        return dict(stride=stride, walk_count=count, nodes=nodes, times=times, lengths=lengths), stats_dict(st)

    def generate(self, edges, mode, cfg: Cfg, thresholds=None, variant=0):
        h = self.build_handle(edges, mode)
        try:
            return self.generate_on(h, cfg, thresholds, variant)
        finally:
            self.L.twref_store_free(h)

    def window_run(self, batches, duration, mode):
        st = I()
        w = self.L.twref_window_create(duration, mode, C.byref(st))
        if not w:
            self._err(st.value)
        try:
            stats = []
            for b in batches:
                e = edges_array(b)
                bs = BatchStatsC()
                rc = self.L.twref_window_ingest(w, _p(e), e.shape[0], C.byref(bs))
                if rc:
                    self._err(rc)
                lo, hi = I64(), I64()
                rcb = self.L.twref_window_bounds(w, C.byref(lo), C.byref(hi))
                stats.append((stats_dict(bs), (lo.value, hi.value) if rcb == 0 else None))
            h = self.L.twref_window_snapshot(w)
            try:
                return stats, self.dump_handle(h)
            finally:
                self.L.twref_store_free(h)
        finally:
            self.L.twref_window_free(w)

    def window_iter(self, batches, duration, mode, keys=None):
        """WindowManager::ingest_batch batch by batch (window_manager.cpp:14-62):
        yields (BatchStats, window_bounds, snapshot dump) after EVERY batch,
        one snapshot at a time (large windows: nothing accumulates)."""
        st = I()
        w = self.L.twref_window_create(duration, mode, C.byref(st))
        if not w:
            self._err(st.value)
        try:
            for b in batches:
                e = edges_array(b)
                bs = BatchStatsC()
                rc = self.L.twref_window_ingest(w, _p(e), e.shape[0], C.byref(bs))
                if rc:
                    self._err(rc)
                lo, hi = I64(), I64()
                rcb = self.L.twref_window_bounds(w, C.byref(lo), C.byref(hi))
                h = self.L.twref_window_snapshot(w)
                try:
                    d = self.dump_handle(h, keys)
                finally:
                    self.L.twref_store_free(h)
                yield stats_dict(bs), ((lo.value, hi.value) if rcb == 0 else None), d
        finally:
            self.L.twref_window_free(w)

    def replay(self, edges, batch_duration, window_duration, mode, cfg: Cfg, thresholds=None, variant=0,
               generate=True):
        e = edges_array(edges)
        c = ReplayCfgRef(batch_duration=batch_duration, window_duration=window_duration, mode=mode,
                         variant=variant, generate=int(generate), keep_walks=1, walk=cfg.c(),
                         thresholds=ThresholdsC(*(thresholds or (4, 256, 8192, 512, 4096))))
        nb = U64()
        st = I()
        h = self.L.twref_replay(_p(e), e.shape[0], C.byref(c), C.byref(nb), C.byref(st))
        if not h:
            self._err(st.value)
        out = []
        try:
            for b in range(nb.value):
                bs, ws = BatchStatsC(), WalkStatsC()
                self.L.twref_replay_record(h, b, C.byref(bs), C.byref(ws))
                w = self.L.twref_replay_walks(h, b)
                stride = self.L.twref_walks_stride(w)
                count = self.L.twref_walks_count(w)
                nodes = np.zeros(count * stride, np.int64)
                times = np.zeros(count * stride, np.int64)
                lengths = np.zeros(count, np.uint32)
                self.L.twref_walks_copy(w, _p(nodes), _p(times), _p(lengths))
                out.append((stats_dict(bs), stats_dict(ws),
                            dict(stride=stride, walk_count=count, nodes=nodes, times=times, lengths=lengths)))
        finally:
            self.L.twref_replay_free(h)
        return out

    def read_edges_tsv(self, text: bytes):
        """read_edges_tsv (io.cpp:40-63): (edges (n, 3) int64, None) or
        (None, (line, what())) on a ParseError."""
        buf = np.frombuffer(text, np.uint8) if text else np.zeros(1, np.uint8)
        n, line = U64(), U64()
        rc = self.L.twref_read_edges_tsv(_p(buf), len(text), None, 0, C.byref(n), C.byref(line))
        if rc == 5:
            return None, (line.value, self.L.twref_last_error().decode())
        if rc:
            self._err(rc)
        out = np.zeros((max(n.value, 1), 3), np.int64)
        rc = self.L.twref_read_edges_tsv(_p(buf), len(text), _p(out), n.value, C.byref(n), C.byref(line))
        if rc:
            self._err(rc)
        return out[: n.value], None

    def write_edges_tsv(self, edges) -> bytes:
        e = edges_array(edges)
        n = U64()
        rc = self.L.twref_write_edges_tsv(_p(e), e.shape[0], None, 0, C.byref(n))
        if rc:
            self._err(rc)
        buf = np.empty(max(n.value, 1), np.uint8)
        rc = self.L.twref_write_edges_tsv(_p(e), e.shape[0], _p(buf), buf.size, C.byref(n))
        if rc:
            self._err(rc)
        return buf[: n.value].tobytes()

    def serialize_walks(self, walks: dict, binary: bool) -> bytes:
        """The reference's write_walks_text / write_walks_binary (io.cpp:119-135, :173-183)."""
        args = (walks["stride"], walks["walk_count"], _p(np.ascontiguousarray(walks["nodes"], np.int64)),
                _p(np.ascontiguousarray(walks["times"], np.int64)),
                _p(np.ascontiguousarray(walks["lengths"], np.uint32)), int(binary))
        n = U64()
        rc = self.L.twref_walks_serialize(*args, None, 0, C.byref(n))
        if rc:
            self._err(rc)
        buf = np.empty(max(n.value, 1), np.uint8)
        rc = self.L.twref_walks_serialize(*args, _p(buf), buf.size, C.byref(n))
        if rc:
            self._err(rc)
        return buf[: n.value].tobytes()

    def check_walkset(self, edges, undirected, walks: dict, direction=0):
        e = edges_array(edges)
        out = np.zeros(4, np.uint64)
        rc = self.L.twref_check_walkset(_p(e), e.shape[0], int(undirected), walks["stride"], walks["walk_count"],
                                        _p(np.ascontiguousarray(walks["nodes"])),
                                        _p(np.ascontiguousarray(walks["times"])),
                                        _p(np.ascontiguousarray(walks["lengths"])), direction, _p(out))
        if rc:
            self._err(rc)
        return tuple(int(x) for x in out)
