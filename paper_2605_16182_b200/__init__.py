"""B200-native streaming temporal random walk engine (arxiv 2605.16182,
"Tempest"), drop-in for the reference `timewalk` core's hot path.

The compute lives in libtimewalk_b200.so (hand-written sm_100a CUDA behind
the C ABI in include/twg.h); this package is the Python mirror of the
reference's public API (see timewalk.py). Importing it loads the library and
fails loudly if it has not been built.
"""
from . import _abi
from .timewalk import *  # noqa: F401,F403
from .timewalk import (BatchRecord, BatchStats, BiasKind, Context, DirectionMode, EdgeStore,  # noqa: F401
                       LogicError, Node2VecParams, ReplayConfig, RngKind, StartMode, TierCounts,
                       TierThresholds, Variant, WalkConfig, WalkDirection, WalkSet, WalkStats, WindowManager,
                       DeviceEdges, default_context, format_edges_tsv, generate_walks, generate_walks_fullwalk, ParseError,
                       read_edges_tsv, replay_stream, sample_start_edge, synth_graph)

_abi.load()
