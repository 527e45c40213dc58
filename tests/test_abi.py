"""CPU-only checks of the drop-in boundary: the C-ABI library loads without a
GPU and exports every symbol include/twg.h declares; struct layouts match
the header; the oracle builds. No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    from paper_2605_16182_b200 import _abi
    lib = _abi.load()
    syms = _abi.header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_abi.SIGNATURES), "ctypes signatures out of sync with include/twg.h"
    assert lib.twg_abi_version() == 1


def test_dynamic_symbol_table():
    from paper_2605_16182_b200 import _abi
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(twg_[a-z_0-9]+)\b", out))
    assert set(_abi.header_symbols()) <= exported


def test_struct_sizes_match_header():
    """Compile a tiny C program against include/twg.h and compare sizeof/offsets with ctypes."""
    from paper_2605_16182_b200 import _abi
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "twg.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(twg_edge), sizeof(twg_walk_config), sizeof(twg_walk_stats),
        sizeof(twg_batch_stats), sizeof(twg_store_info), sizeof(twg_thresholds), sizeof(twg_build_opts));
 printf("%zu %zu %zu\n", offsetof(twg_walk_config, seed), offsetof(twg_walk_config, walk_end),
        offsetof(twg_walk_stats, alg_bytes));
 return 0; }
'''
    d = os.path.join(ROOT, "build")
    os.makedirs(d, exist_ok=True)
    c = os.path.join(d, "abi_sizes.c")
    open(c, "w").write(src)
    exe = os.path.join(d, "abi_sizes")
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
    lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    sizes = [int(x) for x in lines[0].split()]
    assert sizes == [C.sizeof(_abi.twg_edge), C.sizeof(_abi.twg_walk_config), C.sizeof(_abi.twg_walk_stats),
                     C.sizeof(_abi.twg_batch_stats), C.sizeof(_abi.twg_store_info), C.sizeof(_abi.twg_thresholds),
                     C.sizeof(_abi.twg_build_opts)]
    offs = [int(x) for x in lines[1].split()]
    assert offs == [_abi.twg_walk_config.seed.offset, _abi.twg_walk_config.walk_end.offset,
                    _abi.twg_walk_stats.alg_bytes.offset]


def test_kernels_compiled_for_sm100a():
    from paper_2605_16182_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_without_gpu_are_loud():
    """No CPU fallback: a compute call without a usable GPU fails, it does not
    silently run on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_16182_b200 as tw
    with pytest.raises(RuntimeError):
        tw.Context(0)
