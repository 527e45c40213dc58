"""Python mirror of the reference's public `timewalk` API (proj/core), served
by the B200 library through the C ABI (include/twg.h).

Same names, argument meaning, defaults and error behaviour as the C++ API
(edge_store.hpp, window_manager.hpp, walk_engine.hpp, samplers.hpp,
replay.hpp), so the parity tests read like the reference's own tests.
Errors map as the reference's exceptions do:
  std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
  std::logic_error -> LogicError (RuntimeError subclass).
Every computation runs on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _abi

kTimeUnset = -(2**63)
kTimeInfinite = 2**63 - 1
kExponentialExactLimit = 700
kNode2VecMaxRetries = 64


class ParseError(RuntimeError):
    """timewalk::ParseError (io.hpp:15-23): message + 1-based line."""

    def __init__(self, what: str, line: int):
        super().__init__(f"{what} (line {line})")
        self.line = line


class LogicError(RuntimeError):
    """std::logic_error."""


class DirectionMode(enum.IntEnum):
    DirectedForward = 0
    DirectedBackward = 1
    Undirected = 2


class WalkDirection(enum.IntEnum):
    Forward = 0
    Backward = 1


class BiasKind(enum.IntEnum):
    UniformIndex = 0
    LinearIndex = 1
    ExponentialIndex = 2
    ExponentialWeight = 3


class StartMode(enum.IntEnum):
    PerNode = 0
    Sampled = 1


class Variant(enum.IntEnum):
    Coop = 0
    CoopDirect = 1
    FullWalk = 2


class RngKind(enum.IntEnum):
    SplitMix = 0  # the reference's CounterRng (rng.hpp), bit-exact
    Philox = 1    # Philox4x32-10 keyed by (seed; walk, hop, ordinal)


def start_sentinel(direction: WalkDirection) -> int:
    return kTimeUnset if direction == WalkDirection.Forward else kTimeInfinite


# --------------------------------------------------------------------------- errors

def _raise(code: int) -> None:
    lib = _abi.load()
    msg = (lib.twg_last_error() or b"").decode()
    if code == _abi.TWG_EINVAL:
        raise ValueError(msg)
    if code == _abi.TWG_ERANGE:
        raise IndexError(msg)
    if code == _abi.TWG_ELOGIC:
        raise LogicError(msg)
    if code == _abi.TWG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"twg error {code}: {msg}")


def _call(name: str, *args) -> None:
    rc = getattr(_abi.load(), name)(*args)
    if rc != 0:
        _raise(rc)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data) if a.size else C.c_void_p(0)


# --------------------------------------------------------------------------- edge files

class DeviceEdges:
    """A device edge list (twg_edges): the result of the device TSV parser or
    an upload; SoA columns in HBM (``device()`` views feed
    WindowManager.ingest_batch_device directly)."""

    def __init__(self, handle: C.c_void_p):
        self.handle = handle
        n = C.c_uint64()
        _call("twg_edges_info", handle, C.byref(n))
        self.count = n.value

    def __del__(self):
        try:
            if self.handle:
                _abi.load().twg_edges_destroy(self.handle)
        except Exception:
            pass

    @classmethod
    def parse_tsv(cls, text: bytes, ctx: Optional["Context"] = None) -> "DeviceEdges":
        """read_edges_tsv (io.cpp:40-63) on the device. Raises ParseError like the reference."""
        ctx = ctx or default_context()
        buf = np.frombuffer(text, np.uint8) if text else np.zeros(1, np.uint8)
        h, line = C.c_void_p(), C.c_uint64()
        lib = _abi.load()
        rc = lib.twg_parse_edges_tsv(ctx.handle, _ptr(buf), len(text), C.byref(h), C.byref(line))
        if rc == _abi.TWG_EPARSE:
            raise ParseError((lib.twg_last_error() or b"").decode(), line.value)
        if rc:
            _raise(rc)
        return cls(h)

    @classmethod
    def from_array(cls, edges, ctx: Optional["Context"] = None) -> "DeviceEdges":
        ctx = ctx or default_context()
        e = np.ascontiguousarray(np.asarray(edges, np.int64)).reshape(-1, 3)
        h = C.c_void_p()
        _call("twg_edges_from_host", ctx.handle, _ptr(e), e.shape[0], C.byref(h))
        return cls(h)

    def to_array(self) -> np.ndarray:
        out = np.zeros((max(self.count, 1), 3), np.int64)
        _call("twg_edges_download", self.handle, _ptr(out))
        return out[: self.count]

    def device(self):
        """(d_src, d_dst, d_t) device pointers (ints), valid while this object lives."""
        s, d, t = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _call("twg_edges_device", self.handle, C.byref(s), C.byref(d), C.byref(t))
        return s.value, d.value, t.value

    def to_tsv(self) -> bytes:
        """write_edges_tsv (io.cpp:65-69), formatted on the device."""
        n = C.c_uint64()
        _call("twg_edges_format_tsv", self.handle, None, 0, C.byref(n))
        buf = np.empty(max(n.value, 1), np.uint8)
        _call("twg_edges_format_tsv", self.handle, _ptr(buf), buf.size, C.byref(n))
        return buf[: n.value].tobytes()


def synth_graph(kind: str, a: int, b: int = 0, t_max: int = 0, seed: int = 0,
                ctx: Optional["Context"] = None) -> np.ndarray:
    """The reference's synthetic graphs (synthetic.hpp) generated on the GPU,
    bit-identical: kind "uniform" (a nodes, b edges, t_max), "hub_skewed" (a
    background nodes, b background edges), "mega_hub" (a feeders),
    "time_ladder" (a edges, b rungs). Returns (n, 3) int64."""
    k = {"uniform": 0, "hub_skewed": 1, "mega_hub": 2, "time_ladder": 3}[kind]
    ctx = ctx or default_context()
    n = C.c_uint64()
    _call("twg_synth_graph", ctx.handle, k, a, b, t_max, seed, None, 0, C.byref(n))
    out = np.zeros((max(n.value, 1), 3), np.int64)
    _call("twg_synth_graph", ctx.handle, k, a, b, t_max, seed, _ptr(out), n.value, C.byref(n))
    return out[: n.value]


def read_edges_tsv(text: bytes, ctx: Optional["Context"] = None) -> np.ndarray:
    """read_edges_tsv (io.cpp:40-63), parsed on the device: (n, 3) int64."""
    return DeviceEdges.parse_tsv(text, ctx).to_array()


def format_edges_tsv(edges, ctx: Optional["Context"] = None) -> bytes:
    """write_edges_tsv (io.cpp:65-69), formatted on the device."""
    return DeviceEdges.from_array(edges, ctx).to_tsv()


# --------------------------------------------------------------------------- context

class Context:
    """One device + stream + stream-ordered pool (twg_ctx)."""

    def __init__(self, device: int = 0, priority: int = 0):
        h = C.c_void_p()
        _call("twg_ctx_create_prio", device, int(priority), C.byref(h))
        self.handle = h
        self.device = device

    def sync(self) -> None:
        _call("twg_ctx_sync", self.handle)

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _call("twg_ctx_stream", self.handle, C.byref(s))
        return s.value or 0

    @property
    def launches(self) -> int:
        n = C.c_uint64()
        _call("twg_ctx_launch_count", self.handle, C.byref(n))
        return n.value

    def __del__(self):
        try:
            if self.handle:
                _abi.load().twg_ctx_destroy(self.handle)
        except Exception:
            pass


_ctx_lock = threading.Lock()
_contexts: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    with _ctx_lock:
        if device not in _contexts:
            _contexts[device] = Context(device)
        return _contexts[device]


# --------------------------------------------------------------------------- edges

def as_edges(edges) -> np.ndarray:
    """(n, 3) C-contiguous int64 [src, dst, t] == TemporalEdge AoS."""
    if isinstance(edges, np.ndarray):
        a = np.ascontiguousarray(edges, dtype=np.int64)
    else:
        a = np.ascontiguousarray(np.array(list(edges), dtype=np.int64))
    if a.size == 0:
        return np.zeros((0, 3), dtype=np.int64)
    return a.reshape(-1, 3)


@dataclass
class NeighborRange:
    start: int = 0
    end: int = 0
    group_count: int = 0

    def empty(self) -> bool:
        return self.start == self.end

    def size(self) -> int:
        return self.end - self.start


@dataclass
class TsGroupMark:
    time: int
    start: int


# field ids of twg_store_download
_F = dict(src_ext=(0, np.int64, "m"), dst_ext=(1, np.int64, "m"), t=(2, np.int64, "m"),
          src=(3, np.uint32, "m"), dst=(4, np.uint32, "m"), ts_off=(5, np.uint64, "Z1"),
          ts_time=(6, np.int64, "Z"), ts_w=(7, np.float64, "Z"), n_off=(8, np.uint64, "V1"),
          n_tsidx=(9, np.uint64, "V1"), mk_time=(10, np.int64, "Q"), mk_start=(11, np.uint32, "Q"),
          ref_edge=(12, np.uint32, "P"), wprefix=(13, np.float64, "P"), ext=(14, np.int64, "V"),
          ref_nbr=(15, np.uint32, "P"), adj_off=(16, np.uint64, "V1"), adj=(17, np.uint32, "A"))


class EdgeStore:
    """Immutable dual-index snapshot resident on the GPU (edge_store.hpp:167-199).
    Accessors read a lazily downloaded host mirror (the reference's inline
    span accessors, edge_store.hpp:76-145)."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        self._mirror: dict[str, np.ndarray] = {}
        self._refresh_info()

    def _refresh_info(self):
        info = _abi.twg_store_info()
        _call("twg_store_get_info", self.handle, C.byref(info))
        self.info = info

    def __del__(self):
        try:
            if self.handle:
                _abi.load().twg_store_release(self.handle)
        except Exception:
            pass

    @staticmethod
    def build(edges, mode: DirectionMode = DirectionMode.DirectedForward, *, weights: bool = True,
              adjacency: bool = True, ctx: Optional[Context] = None) -> "EdgeStore":
        ctx = ctx or default_context()
        e = as_edges(edges)
        opts = _abi.twg_build_opts(int(weights), int(adjacency))
        h = C.c_void_p()
        _call("twg_store_build", ctx.handle, _ptr(e), e.shape[0], int(mode), C.byref(opts), C.byref(h))
        return EdgeStore(h, ctx)

    # --- raw arrays -----------------------------------------------------------------
    def array(self, name: str) -> np.ndarray:
        if name not in self._mirror:
            fid, dt, size = _F[name]
            if name == "adj" or name in ("ts_w", "wprefix"):
                # may be built lazily by the download; refresh counts after
                pass
            i = self.info
            n = {"m": i.edges, "Z": i.ts_groups, "Z1": i.ts_groups + 1, "V": i.nodes, "V1": i.nodes + 1,
                 "Q": i.node_groups, "P": i.entries, "A": None}[size]
            if name == "adj":
                self.array("adj_off")
                self._refresh_info()
                n = self.info.adjacency
            out = np.zeros(max(n, 1), dtype=dt)
            _call("twg_store_download", self.handle, fid, _ptr(out))
            self._mirror[name] = out[:n]
            self._refresh_info()
        return self._mirror[name]

    def dump(self, names=None) -> dict:
        names = names or list(_F)
        return {k: self.array(k) for k in names}

    # --- counts ----------------------------------------------------------------------
    def edge_count(self) -> int:
        return int(self.info.edges)

    def node_count(self) -> int:
        return int(self.info.nodes)

    def is_streaming(self) -> bool:
        """True when the snapshot is a slice of the window's append log / node
        arena (the time-ordered streaming fast path, csrc/append.cu)."""
        return bool(self.info.streaming)

    def layout(self) -> dict:
        """Streaming-representation layout (twg_store_get_layout): log ring,
        arena, rings relocated by the producing ingest, largest ring end."""
        lo = _abi.twg_store_layout()
        _call("twg_store_get_layout", self.handle, C.byref(lo))
        return {n: int(getattr(lo, n)) for n, _ in lo._fields_}

    def ts_group_count(self) -> int:
        return int(self.info.ts_groups)

    def empty(self) -> bool:
        return self.info.edges == 0

    def direction_mode(self) -> DirectionMode:
        return DirectionMode(self.info.mode)

    def supports(self, d: WalkDirection) -> bool:
        if self.info.mode == DirectionMode.Undirected:
            return True
        return (self.info.mode == DirectionMode.DirectedForward) == (d == WalkDirection.Forward)

    def memory_bytes(self) -> int:
        return int(self.info.device_bytes)

    # --- timestamp-grouped view ------------------------------------------------------
    def edge_slice_for_ts_group(self, g: int) -> tuple[int, int]:
        if g < 0 or g >= self.ts_group_count():
            raise IndexError("edge_slice_for_ts_group: group index out of range")
        off = self.array("ts_off")
        return int(off[g]), int(off[g + 1])

    def ts_group_time(self, g: int) -> int:
        return int(self.array("ts_time")[g])

    def ts_group_weight_prefix(self) -> np.ndarray:
        return self.array("ts_w")

    def edge_at(self, pos: int) -> tuple[int, int, int]:
        return (int(self.array("src_ext")[pos]), int(self.array("dst_ext")[pos]), int(self.array("t")[pos]))

    def edge_source_internal(self, pos: int) -> int:
        return int(self.array("src")[pos])

    def edge_target_internal(self, pos: int) -> int:
        return int(self.array("dst")[pos])

    def edge_time(self, pos: int) -> int:
        return int(self.array("t")[pos])

    def edge_times(self) -> np.ndarray:
        return self.array("t")

    # --- node ids ----------------------------------------------------------------------
    def find_nodes(self, ext) -> tuple[np.ndarray, np.ndarray]:
        v = np.ascontiguousarray(np.asarray(ext, dtype=np.int64).reshape(-1))
        internal = np.zeros(max(v.size, 1), np.uint32)
        found = np.zeros(max(v.size, 1), np.uint8)
        _call("twg_store_find_nodes", self.handle, _ptr(v), v.size, _ptr(internal), _ptr(found))
        return internal[: v.size], found[: v.size].astype(bool)

    def find_node(self, ext: int) -> Optional[int]:
        i, f = self.find_nodes([ext])
        return int(i[0]) if f[0] else None

    def external_id(self, v: int) -> int:
        return int(self.array("ext")[v])

    # --- node-and-timestamp-grouped view ------------------------------------------------
    def temporal_neighborhoods(self, v_ext, t, direction: WalkDirection) -> np.ndarray:
        v = np.ascontiguousarray(np.asarray(v_ext, dtype=np.int64).reshape(-1))
        tt = np.ascontiguousarray(np.broadcast_to(np.asarray(t, dtype=np.int64), v.shape))
        out = np.zeros((max(v.size, 1), 3), np.uint64)
        _call("twg_store_neighborhood", self.handle, _ptr(v), _ptr(tt), v.size, int(direction), _ptr(out))
        return out[: v.size]

    def temporal_neighborhood(self, v: int, t: int, direction: WalkDirection) -> NeighborRange:
        r = self.temporal_neighborhoods([v], [t], direction)[0]
        return NeighborRange(int(r[0]), int(r[1]), int(r[2]))

    def temporal_neighborhood_internal(self, v: int, t: int, direction: WalkDirection) -> NeighborRange:
        return self.temporal_neighborhood(self.external_id(v), t, direction)

    def timestamp_group_count(self, v_ext: int) -> int:
        iv = self.find_node(v_ext)
        return 0 if iv is None else self.timestamp_group_count_internal(iv)

    def timestamp_group_count_internal(self, v: int) -> int:
        ti = self.array("n_tsidx")
        return int(ti[v + 1] - ti[v])

    def node_region(self, v: int) -> tuple[int, int]:
        off = self.array("n_off")
        return int(off[v]), int(off[v + 1])

    def group_marks(self, v: int) -> list[TsGroupMark]:
        ti = self.array("n_tsidx")
        mt, ms = self.array("mk_time"), self.array("mk_start")
        return [TsGroupMark(int(mt[g]), int(ms[g])) for g in range(int(ti[v]), int(ti[v + 1]))]

    def ref_edge(self, pos: int) -> int:
        return int(self.array("ref_edge")[pos])

    def ref_time(self, pos: int) -> int:
        return int(self.array("t")[self.array("ref_edge")[pos]])

    def ref_neighbor(self, pos: int, owner: int) -> int:
        e = self.ref_edge(pos)
        src, dst = self.array("src"), self.array("dst")
        if self.info.mode == DirectionMode.DirectedForward:
            return int(dst[e])
        if self.info.mode == DirectionMode.DirectedBackward:
            return int(src[e])
        return int(dst[e]) if src[e] == owner else int(src[e])

    def weight_prefix(self) -> np.ndarray:
        return self.array("wprefix")

    # --- adjacency -------------------------------------------------------------------------
    def adjacent_many(self, a, b, temporal: bool = False, t=None,
                      direction: WalkDirection = WalkDirection.Forward) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.uint32).reshape(-1))
        b = np.ascontiguousarray(np.asarray(b, dtype=np.uint32).reshape(-1))
        tt = np.ascontiguousarray(np.broadcast_to(np.asarray(0 if t is None else t, dtype=np.int64), a.shape))
        out = np.zeros(max(a.size, 1), np.uint8)
        _call("twg_store_adjacent", self.handle, _ptr(a), _ptr(b), a.size, int(temporal), _ptr(tt),
              int(direction), _ptr(out))
        return out[: a.size].astype(bool)

    def adjacent(self, a: int, b: int) -> bool:
        return bool(self.adjacent_many([a], [b])[0])

    def adjacent_after(self, a: int, b: int, t: int, direction: WalkDirection) -> bool:
        return bool(self.adjacent_many([a], [b], True, [t], direction)[0])

    # --- maintenance --------------------------------------------------------------------------
    def export_suffix(self, cutoff: int) -> np.ndarray:
        t = self.array("t")
        lo = int(np.searchsorted(t, cutoff, side="left"))
        return np.stack([self.array("src_ext")[lo:], self.array("dst_ext")[lo:], t[lo:]], axis=1)

    def export_edges(self) -> np.ndarray:
        return self.export_suffix(kTimeUnset)


# --------------------------------------------------------------------------- window

@dataclass
class BatchStats:
    ingested: int = 0
    dropped_late: int = 0
    evicted: int = 0
    retained: int = 0
    rebuild_duration: float = 0.0
    peak_bytes: int = 0

    @staticmethod
    def of(s: _abi.twg_batch_stats) -> "BatchStats":
        return BatchStats(s.ingested, s.dropped_late, s.evicted, s.retained, s.rebuild_duration, s.peak_bytes)


class WindowManager:
    """Sliding window (window_manager.hpp:31-62), device-resident."""

    def __init__(self, duration: int, mode: DirectionMode = DirectionMode.DirectedForward, *,
                 weights: bool = True, adjacency: bool = True, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        opts = _abi.twg_build_opts(int(weights), int(adjacency))
        h = C.c_void_p()
        _call("twg_window_create", self.ctx.handle, int(duration), int(mode), C.byref(opts), C.byref(h))
        self.handle = h
        self.duration = int(duration)

    def __del__(self):
        try:
            if self.handle:
                _abi.load().twg_window_destroy(self.handle)
        except Exception:
            pass

    def ingest_batch(self, batch) -> BatchStats:
        e = as_edges(batch)
        st = _abi.twg_batch_stats()
        _call("twg_window_ingest", self.handle, _ptr(e), e.shape[0], C.byref(st))
        return BatchStats.of(st)

    def ingest_batch_device(self, d_src: int, d_dst: int, d_t: int, n: int, stats: bool = True):
        st = _abi.twg_batch_stats()
        _call("twg_window_ingest_device", self.handle, C.c_void_p(d_src), C.c_void_p(d_dst), C.c_void_p(d_t), n,
              C.byref(st) if stats else None)
        return BatchStats.of(st) if stats else None

    def snapshot(self) -> EdgeStore:
        h = C.c_void_p()
        _call("twg_window_snapshot", self.handle, C.byref(h))
        return EdgeStore(h, self.ctx)

    def window_bounds(self) -> tuple[int, int]:
        lo, hi = C.c_int64(), C.c_int64()
        _call("twg_window_bounds", self.handle, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def _state(self):
        th, bc, st = C.c_int64(), C.c_uint64(), _abi.twg_batch_stats()
        _call("twg_window_state", self.handle, C.byref(th), C.byref(bc), C.byref(st))
        return th.value, bc.value, st

    def t_high(self) -> int:
        return self._state()[0]

    def batch_count(self) -> int:
        return self._state()[1]

    def last_batch_stats(self) -> BatchStats:
        return BatchStats.of(self._state()[2])

    def cutoff_for(self, high: int) -> int:
        return high - self.duration if high > self.duration else 0


# --------------------------------------------------------------------------- walks

@dataclass
class TierThresholds:
    w_warp: int = 4
    block_dim: int = 256
    w_max: int = 8192
    g_warp_cap: int = 512
    g_block_cap: int = 4096

    def validate(self) -> None:
        if self.w_warp < 1 or self.w_warp > self.block_dim or self.block_dim > self.w_max:
            raise ValueError("tier thresholds: need 1 <= w_warp <= block_dim <= w_max")
        if self.g_warp_cap > self.g_block_cap:
            raise ValueError("tier thresholds: need g_warp_cap <= g_block_cap")

    def c(self) -> _abi.twg_thresholds:
        return _abi.twg_thresholds(self.w_warp, self.block_dim, self.w_max, self.g_warp_cap, self.g_block_cap)


@dataclass
class Node2VecParams:
    p: float = 1.0
    q: float = 1.0

    def beta_max(self) -> float:
        return max(1.0 / self.p, 1.0, 1.0 / self.q)


@dataclass
class WalkConfig:
    walk_length: int = 80
    start_mode: StartMode = StartMode.PerNode
    walks_per_node: int = 10
    total_walks: int = 0
    bias: BiasKind = BiasKind.ExponentialWeight
    start_bias: BiasKind = BiasKind.UniformIndex
    node2vec: Optional[Node2VecParams] = None
    node2vec_temporal_adjacency: bool = False
    direction: WalkDirection = WalkDirection.Forward
    seed: int = 0
    rng: RngKind = RngKind.SplitMix
    walk_begin: int = 0  # shard of the global walk-id space (0, 0 = all)
    walk_end: int = 0

    def validate(self) -> None:
        if self.walk_length < 1:
            raise ValueError("walk config: walk_length must be >= 1")
        if self.start_mode == StartMode.PerNode and self.walks_per_node == 0:
            raise ValueError("walk config: walks_per_node must be positive")
        if self.node2vec and (self.node2vec.p <= 0.0 or self.node2vec.q <= 0.0):
            raise ValueError("walk config: node2vec p and q must be positive")

    def c(self) -> _abi.twg_walk_config:
        n2v = self.node2vec
        return _abi.twg_walk_config(
            walk_length=self.walk_length, start_mode=int(self.start_mode), walks_per_node=self.walks_per_node,
            total_walks=self.total_walks, bias=int(self.bias), start_bias=int(self.start_bias),
            node2vec=1 if n2v else 0, temporal_adjacency=int(self.node2vec_temporal_adjacency),
            p=n2v.p if n2v else 1.0, q=n2v.q if n2v else 1.0, direction=int(self.direction),
            rng=int(self.rng), seed=self.seed, walk_begin=self.walk_begin, walk_end=self.walk_end)


@dataclass
class TierCounts:
    solo: int = 0
    warp_cached: int = 0
    warp_direct: int = 0
    block_cached: int = 0
    block_direct: int = 0
    multi_block: int = 0

    def total(self) -> int:
        return self.solo + self.warp_cached + self.warp_direct + self.block_cached + self.block_direct + \
            self.multi_block


@dataclass
class WalkStats:
    walks: int = 0
    hops: int = 0
    steps: int = 0
    tiers: TierCounts = field(default_factory=TierCounts)
    wall_seconds: float = 0.0
    ambiguous_draws: int = 0
    alg_bytes: int = 0

    def fill(self, s: _abi.twg_walk_stats) -> None:
        self.walks, self.hops, self.steps = s.walks, s.hops, s.steps
        self.tiers = TierCounts(s.solo, s.warp_cached, s.warp_direct, s.block_cached, s.block_direct,
                                s.multi_block)
        self.wall_seconds = s.wall_seconds
        self.ambiguous_draws = s.ambiguous_draws
        self.alg_bytes = s.alg_bytes


class WalkSet:
    """Fixed-stride walks (walk_engine.hpp:55-70). Device-resident until a
    host array is requested."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        stride, count, first, hops = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _call("twg_walkset_info", handle, C.byref(stride), C.byref(count), C.byref(first), C.byref(hops))
        self.stride = stride.value
        self.walk_count = count.value
        self.first_walk = first.value
        self.total_hops = hops.value
        self._nodes = self._times = self._lengths = None

    def __del__(self):
        try:
            if self.handle:
                _abi.load().twg_walkset_destroy(self.handle)
        except Exception:
            pass

    def audit(self, store: "EdgeStore", direction: WalkDirection = WalkDirection.Forward, strict: bool = True,
              first_violation: bool = False):
        """Causality audit on the GPU (validity.cpp:108-120 check_walkset):
        returns (report dict, per-walk first invalid hop or -1 | None)."""
        rep = _abi.twg_audit_report()
        fv = np.zeros(max(self.walk_count, 1), np.int64) if first_violation else None
        _call("twg_walkset_audit", self.handle, store.handle, int(direction), int(strict),
              _ptr(fv) if fv is not None else None, C.byref(rep))
        out = {"walks": rep.walks, "valid_walks": rep.valid_walks, "hops": rep.hops, "valid_hops": rep.valid_hops}
        return out, (fv[: self.walk_count] if fv is not None else None)

    @classmethod
    def from_arrays(cls, stride: int, nodes, times, lengths, ctx: Optional[Context] = None) -> "WalkSet":
        """A device walk set from a host WalkSet image (walk-major nodes /
        times of walk_count x stride, lengths) — e.g. walks of another engine
        to be written with the writers below."""
        ctx = ctx or default_context()
        lengths = np.ascontiguousarray(lengths, np.uint32)
        nodes = np.ascontiguousarray(nodes, np.int64).reshape(-1)
        times = np.ascontiguousarray(times, np.int64).reshape(-1)
        count = len(lengths)
        if nodes.size != count * stride or times.size != count * stride:
            raise ValueError("WalkSet.from_arrays: nodes/times must hold walk_count * stride entries")
        h = C.c_void_p()
        _call("twg_walkset_from_host", ctx.handle, int(stride), count, _ptr(nodes), _ptr(times), _ptr(lengths),
              C.byref(h))
        return cls(h, ctx)

    def to_text(self) -> bytes:
        """write_walks_text (io.cpp:119-135), formatted on the device."""
        n = C.c_uint64()
        _call("twg_walkset_text", self.handle, None, 0, C.byref(n))
        buf = np.empty(max(n.value, 1), np.uint8)
        _call("twg_walkset_text", self.handle, _ptr(buf), buf.size, C.byref(n))
        return buf[: n.value].tobytes()

    def to_binary(self) -> bytes:
        """write_walks_binary (io.cpp:173-183): the TMPW0002 image."""
        n = C.c_uint64()
        _call("twg_walkset_binary", self.handle, None, 0, C.byref(n))
        buf = np.empty(max(n.value, 1), np.uint8)
        _call("twg_walkset_binary", self.handle, _ptr(buf), buf.size, C.byref(n))
        return buf[: n.value].tobytes()

    def write(self, path: str, binary: bool = False) -> None:
        """write_walks (io.hpp:61): the text or binary image to a file."""
        with open(path, "wb") as f:
            f.write(self.to_binary() if binary else self.to_text())

    def _download(self):
        if self._nodes is None:
            cells = self.walk_count * self.stride
            n = np.zeros(max(cells, 1), np.int64)
            t = np.zeros(max(cells, 1), np.int64)
            ln = np.zeros(max(self.walk_count, 1), np.uint32)
            _call("twg_walkset_download", self.handle, _ptr(n), _ptr(t), _ptr(ln))
            self._nodes, self._times, self._lengths = n[:cells], t[:cells], ln[: self.walk_count]

    @property
    def nodes(self) -> np.ndarray:
        self._download()
        return self._nodes

    @property
    def times(self) -> np.ndarray:
        self._download()
        return self._times

    @property
    def lengths(self) -> np.ndarray:
        if self._lengths is None:
            ln = np.zeros(max(self.walk_count, 1), np.uint32)
            _call("twg_walkset_download", self.handle, None, None, _ptr(ln))
            self._lengths = ln[: self.walk_count]
        return self._lengths

    def compact(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(offsets[count+1], nodes[total], times[total]) — recorded entries only."""
        lengths = self.lengths.astype(np.uint64)
        total = int(lengths.sum())
        offs = np.zeros(self.walk_count + 1, np.uint64)
        n = np.zeros(max(total, 1), np.int64)
        t = np.zeros(max(total, 1), np.int64)
        _call("twg_walkset_download_compact", self.handle, _ptr(offs), _ptr(n), _ptr(t))
        return offs, n[:total], t[:total]

    def node_at(self, walk: int, slot: int) -> int:
        return int(self.nodes[walk * self.stride + slot])

    def time_at(self, walk: int, slot: int) -> int:
        return int(self.times[walk * self.stride + slot])

    def __eq__(self, other) -> bool:
        return (self.stride == other.stride and self.walk_count == other.walk_count and
                np.array_equal(self.nodes, other.nodes) and np.array_equal(self.times, other.times) and
                np.array_equal(self.lengths, other.lengths))


def generate_walks(store: EdgeStore, config: WalkConfig, thresholds: Optional[TierThresholds] = None,
                   variant: Variant = Variant.Coop, stats: Optional[WalkStats] = None,
                   ctx: Optional[Context] = None) -> WalkSet:
    """walk_engine.hpp:165-167. ctx: run on another context's stream (e.g. a
    walk stream overlapping the next batch's ingest; the window protects the
    current and the retired snapshot while it ingests)."""
    ctx = ctx or store.ctx
    th = (thresholds or TierThresholds()).c()
    cfg = config.c()
    h = C.c_void_p()
    st = _abi.twg_walk_stats()
    _call("twg_generate", ctx.handle, store.handle, C.byref(cfg), C.byref(th), int(variant), C.byref(h),
          C.byref(st))
    if stats is not None:
        stats.fill(st)
    return WalkSet(h, ctx)


def generate_walks_fullwalk(store: EdgeStore, config: WalkConfig, stats: Optional[WalkStats] = None) -> WalkSet:
    return generate_walks(store, config, TierThresholds(), Variant.FullWalk, stats)


@dataclass
class GroupBatchStats:
    local: BatchStats
    replica_hash: int
    replicas_agree: bool
    wire_bytes_per_edge: int
    edges: int


def _load_process_nccl() -> None:
    """The group resolves NCCL at run time and uses the copy already loaded
    in the process; when PyTorch is importable it is imported first, so that
    copy is PyTorch's own (two NCCLs cannot share the libnccl.so.2 soname)."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def group_unique_id() -> bytes:
    """The rendezvous id of a ReplicaGroup (ncclUniqueId): one rank creates
    it and shares it out of band (e.g. a torch.distributed broadcast)."""
    _load_process_nccl()
    buf = (C.c_uint8 * 128)()
    _call("twg_group_unique_id", C.cast(buf, C.c_void_p))
    return bytes(buf)


class ReplicaGroup:
    """Multi-GPU replica group (include/twg.h): one process per
    GPU; batches are broadcast once over NVLink (NCCL) into every rank's
    replica window; walks are sharded by global walk id. Every rank calls
    every method, in the same order."""

    def __init__(self, ctx: Context, nranks: int, rank: int, uid: bytes):
        assert len(uid) == 128
        _load_process_nccl()
        self.ctx = ctx
        self.nranks, self.rank = int(nranks), int(rank)
        ub = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _call("twg_group_create", ctx.handle, self.nranks, self.rank, C.cast(ub, C.c_void_p), C.byref(h))
        self.handle = h

    def close(self) -> None:
        if self.handle:
            _abi.load().twg_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stats(st) -> GroupBatchStats:
        return GroupBatchStats(BatchStats.of(st.local), int(st.replica_hash), bool(st.replicas_agree),
                               int(st.wire_bytes_per_edge), int(st.edges))

    def stage_device(self, slot: int, root: int, d_src: int = 0, d_dst: int = 0, d_t: int = 0, n: int = 0) -> None:
        _call("twg_group_stage_device", self.handle, slot, root, C.c_void_p(d_src), C.c_void_p(d_dst),
              C.c_void_p(d_t), n)

    def stage_host(self, slot: int, root: int, batch=None) -> None:
        if batch is None:
            _call("twg_group_stage_host", self.handle, slot, root, None, 0)
            return
        e = as_edges(batch)
        self._keep = getattr(self, "_keep", {})
        self._keep[slot] = e  # the H2D reads it asynchronously
        _call("twg_group_stage_host", self.handle, slot, root, _ptr(e), e.shape[0])

    def ingest_staged(self, window: WindowManager, slot: int) -> GroupBatchStats:
        st = _abi.twg_group_batch_stats()
        _call("twg_group_ingest_staged", self.handle, window.handle, slot, C.byref(st))
        return self._stats(st)

    def ingest(self, window: WindowManager, root: int, batch=None) -> GroupBatchStats:
        """Root passes the host batch; the other ranks pass None."""
        st = _abi.twg_group_batch_stats()
        if batch is None:
            _call("twg_group_ingest", self.handle, window.handle, root, None, 0, C.byref(st))
        else:
            e = as_edges(batch)
            _call("twg_group_ingest", self.handle, window.handle, root, _ptr(e), e.shape[0], C.byref(st))
        return self._stats(st)

    def ingest_device(self, window: WindowManager, root: int, d_src: int = 0, d_dst: int = 0, d_t: int = 0,
                      n: int = 0) -> GroupBatchStats:
        st = _abi.twg_group_batch_stats()
        _call("twg_group_ingest_device", self.handle, window.handle, root, C.c_void_p(d_src), C.c_void_p(d_dst),
              C.c_void_p(d_t), n, C.byref(st))
        return self._stats(st)

    def generate(self, store: EdgeStore, config: WalkConfig, thresholds: Optional[TierThresholds] = None,
                 variant: Variant = Variant.Coop, stats: Optional[WalkStats] = None,
                 global_stats: Optional[WalkStats] = None) -> WalkSet:
        """This rank's shard of generate_walks (contiguous slice of the global
        walk-id range)."""
        th = (thresholds or TierThresholds()).c()
        cfg = config.c()
        h = C.c_void_p()
        st, gs = _abi.twg_walk_stats(), _abi.twg_walk_stats()
        _call("twg_group_generate", self.handle, store.handle, C.byref(cfg), C.byref(th), int(variant),
              C.byref(h), C.byref(st), C.byref(gs) if global_stats is not None else None)
        if stats is not None:
            stats.fill(st)
        if global_stats is not None:
            global_stats.fill(gs)
        return WalkSet(h, self.ctx)


def replica_hash(store: EdgeStore, tail: int = 0) -> int:
    """The snapshot hash a ReplicaGroup all-reduces after each batch."""
    h = C.c_uint64()
    _call("twg_store_replica_hash", store.handle, int(tail), C.byref(h))
    return h.value


def sample_start_edges(store: EdgeStore, bias: BiasKind, u1, u2) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(u1, dtype=np.float64).reshape(-1))
    b = np.ascontiguousarray(np.asarray(u2, dtype=np.float64).reshape(-1))
    out = np.zeros(max(a.size, 1), np.uint64)
    _call("twg_sample_start_edges", store.handle, int(bias), _ptr(a), _ptr(b), a.size, _ptr(out))
    return out[: a.size]


def sample_start_edge(store: EdgeStore, bias: BiasKind, u1: float, u2: float) -> int:
    """walk_engine.hpp:159."""
    return int(sample_start_edges(store, bias, [u1], [u2])[0])


@dataclass
class DispatchTask:
    node: int
    tier: int
    begin: int
    end: int
    sub_task_index: int = 0
    sub_task_count: int = 1


@dataclass
class StepPlan:
    walk_ids: list
    solo: list
    warp_cached: list
    warp_direct: list
    block_cached: list
    block_direct: list

    def empty(self) -> bool:
        return not (self.solo or self.warp_cached or self.warp_direct or self.block_cached or self.block_direct)


def schedule_step(store: EdgeStore, current, alive, thresholds: Optional[TierThresholds] = None) -> StepPlan:
    """schedule_step over an explicit population (walk_engine.hpp:143-144)."""
    cur = np.ascontiguousarray(np.asarray(current, dtype=np.uint32).reshape(-1))
    al = np.ascontiguousarray(np.asarray(alive, dtype=np.uint8).reshape(-1))
    th = (thresholds or TierThresholds()).c()
    sizes = np.zeros(5, np.uint64)
    cap = cur.size + 16
    rows = np.zeros((cap, 6), np.uint32)
    ids = np.zeros(max(cur.size, 1), np.uint32)
    _call("twg_schedule_step", store.handle, _ptr(cur), _ptr(al), cur.size, C.byref(th), _ptr(sizes), _ptr(rows),
          cap, _ptr(ids))
    lists, r = [], 0
    for k in range(5):
        lst = []
        for _ in range(int(sizes[k])):
            node, b, e, sub, cnt, tier = (int(x) for x in rows[r])
            lst.append(DispatchTask(node, tier, b, e, sub, cnt))
            r += 1
        lists.append(lst)
    n_alive = int(al.astype(bool).sum())
    return StepPlan(list(ids[:n_alive]), *lists)


# --------------------------------------------------------------------------- samplers

def _pick(kind: int, u, n) -> np.ndarray:
    uu = np.ascontiguousarray(np.asarray(u, dtype=np.float64).reshape(-1))
    nn = np.ascontiguousarray(np.broadcast_to(np.asarray(n, dtype=np.uint64), uu.shape))
    out = np.zeros(max(uu.size, 1), np.uint64)
    _call("twg_pick_index", default_context().handle, kind, _ptr(uu), _ptr(nn), uu.size, _ptr(out))
    return out[: uu.size]


def pick_index_uniform(u, n):
    r = _pick(0, u, n)
    return int(r[0]) if np.isscalar(u) else r


def pick_index_linear(u, n):
    r = _pick(1, u, n)
    return int(r[0]) if np.isscalar(u) else r


def pick_index_exponential(u, n):
    r = _pick(2, u, n)
    return int(r[0]) if np.isscalar(u) else r


def pick_weighted_range(u, prefix, begin, end, base):
    pf = np.ascontiguousarray(np.asarray(prefix, dtype=np.float64))
    uu = np.ascontiguousarray(np.atleast_1d(np.asarray(u, dtype=np.float64)))
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(begin, dtype=np.uint64), uu.shape))
    e = np.ascontiguousarray(np.broadcast_to(np.asarray(end, dtype=np.uint64), uu.shape))
    bs = np.ascontiguousarray(np.broadcast_to(np.asarray(base, dtype=np.float64), uu.shape))
    out = np.zeros(max(uu.size, 1), np.uint64)
    _call("twg_pick_weighted_range", default_context().handle, _ptr(uu), _ptr(pf), pf.size, _ptr(b), _ptr(e),
          _ptr(bs), uu.size, _ptr(out))
    return int(out[0]) if np.isscalar(u) else out[: uu.size]


def rng_bits(rng: RngKind, seed: int, walk, hop, ordinal) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(walk, dtype=np.uint64).reshape(-1))
    h = np.ascontiguousarray(np.broadcast_to(np.asarray(hop, dtype=np.uint64), w.shape))
    o = np.ascontiguousarray(np.broadcast_to(np.asarray(ordinal, dtype=np.uint64), w.shape))
    out = np.zeros(max(w.size, 1), np.uint64)
    _call("twg_rng_bits", default_context().handle, int(rng), seed, _ptr(w), _ptr(h), _ptr(o), w.size, _ptr(out))
    return out[: w.size]


# --------------------------------------------------------------------------- replay

@dataclass
class ReplayConfig:
    batch_duration: int = 0
    window_duration: int = 0
    mode: DirectionMode = DirectionMode.DirectedForward
    walk: WalkConfig = field(default_factory=WalkConfig)
    thresholds: TierThresholds = field(default_factory=TierThresholds)
    variant: Variant = Variant.Coop
    generate: bool = True

    def validate(self) -> None:
        if self.batch_duration <= 0:
            raise ValueError("replay: batch_duration must be positive")
        if self.window_duration < self.batch_duration:
            raise ValueError("replay: window_duration must be >= batch_duration")
        self.walk.validate()
        self.thresholds.validate()


@dataclass
class BatchRecord:
    batch_index: int = 0
    ingest: BatchStats = field(default_factory=BatchStats)
    walk: WalkStats = field(default_factory=WalkStats)


def split_batches(times: np.ndarray, batch_duration: int) -> list[tuple[int, int]]:
    """replay.cpp:42-51 batching: spans anchored at the first edge, jumping
    gaps; late edges stay in the current batch. Returns [begin, end) slices."""
    n = times.size
    if n == 0:
        return []
    origin = int(times[0])
    boundary = origin + batch_duration
    out, begin = [], 0
    for i in range(n):
        ti = int(times[i])
        if ti >= boundary:
            if i > begin:
                out.append((begin, i))
                begin = i
            spans = (ti - origin) // batch_duration + 1 if ti >= origin else 1
            boundary = origin + spans * batch_duration
    out.append((begin, n))
    return out


def replay_stream(edges, config: ReplayConfig,
                  sink: Optional[Callable[[BatchRecord, Optional[WalkSet]], None]] = None,
                  ctx: Optional[Context] = None) -> int:
    """replay.hpp:36-37 / replay.cpp:16-53."""
    config.validate()
    e = as_edges(edges)
    if e.shape[0] == 0:
        return 0
    win = WindowManager(config.window_duration, config.mode, ctx=ctx)
    count = 0
    for b, (lo, hi) in enumerate(split_batches(e[:, 2], config.batch_duration)):
        rec = BatchRecord(batch_index=b)
        rec.ingest = win.ingest_batch(e[lo:hi])
        walks = None
        snap = win.snapshot()
        if config.generate and not snap.empty():
            walks = generate_walks(snap, config.walk, config.thresholds, config.variant, rec.walk)
        if sink:
            sink(rec, walks)
        count += 1
    return count
