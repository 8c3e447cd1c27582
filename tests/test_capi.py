"""CPU: the C-ABI library loads and exports every entry point the public
headers declare; host-side validation (which never touches the GPU) follows
the reference's error precedence (kernels.hpp:24-30, error.hpp:8-25)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_1805_02867_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "osmx_b200.h"


def declared_functions() -> set[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return set(re.findall(r"\b(osmx_\w+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (osmx_\w+)", nm))
    missing = names - exported
    assert not missing, f"declared but not exported: {missing}"
    for n in names:
        assert hasattr(lib, n)
    # every declared function has a ctypes signature (and nothing extra)
    assert names == set(_lib.SIGNATURES)


def test_no_torch_or_cxx_types_in_abi():
    raw = HEADER.read_text()
    assert 'extern "C"' in raw
    code = re.sub(r"/\*.*?\*/", "", raw, flags=re.S)  # declarations only
    for bad in ("torch", "std::", "at::", "Tensor", "cudaStream_t"):
        assert bad not in code


def test_cuda_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    # TMA bulk copy (cp.async.bulk -> UBLKCP) and MUFU.EX2 are in the SASS
    assert "UBLKCP" in sass
    assert "MUFU.EX2" in sass


def test_status_strings_and_version():
    lib = _lib.load()
    assert lib.osmx_version() == 100
    assert lib.osmx_status_string(1) == b"empty input vector"  # error.hpp:9
    assert lib.osmx_status_string(2) == b"non-finite input element"  # :14
    assert lib.osmx_status_string(3) == b"k must satisfy 1 <= k <= input size"  # :19
    assert lib.osmx_status_string(4) == b"chunk length must be >= 1"  # :24


def test_validation_without_gpu():
    """Argument errors return synchronously, before any device work."""
    lib = _lib.load()
    fake = C.c_void_p(0x1000)  # never dereferenced: validation fails first
    ws = C.c_void_p(0x2000)
    # V == 0 -> empty_input_error before anything else (kernels.hpp:24-26)
    assert lib.osmx_softmax(2, fake, 0, fake, 0, 4, 0, ws, 1 << 20, None) == _lib.ERR_EMPTY
    assert lib.osmx_softmax_topk(5, fake, 0, 4, 0, 0, fake, fake, ws, 1 << 20, None) == _lib.ERR_EMPTY
    # k out of [1, V] -> invalid_k_error, checked after emptiness (:28-30)
    assert lib.osmx_softmax_topk(5, fake, 10, 4, 10, 0, fake, fake, ws, 1 << 20, None) == _lib.ERR_INVALID_K
    assert lib.osmx_softmax_topk(5, fake, 10, 4, 10, 11, fake, fake, ws, 1 << 20, None) == _lib.ERR_INVALID_K
    assert lib.osmx_topk(fake, 10, 4, 10, 11, fake, fake, ws, 1 << 20, None) == _lib.ERR_INVALID_K
    # device path limits: large-k top-K needs rows * k < 2^31; records k <= OSMX_MAX_K
    assert lib.osmx_softmax_topk(5, fake, 4096, 1 << 20, 4096, 4096, fake, fake, ws, 1 << 20,
                                 None) == _lib.ERR_UNSUPPORTED
    assert lib.osmx_slice_record(fake, 100, 0, 33, fake, ws, 1 << 20, None) == _lib.ERR_UNSUPPORTED
    # bad algorithm id / ld < V / null pointers / small workspace
    assert lib.osmx_softmax(9, fake, 10, fake, 10, 4, 10, ws, 1 << 20, None) == _lib.ERR_INVALID_ARG
    assert lib.osmx_softmax(2, fake, 5, fake, 10, 4, 10, ws, 1 << 20, None) == _lib.ERR_INVALID_ARG
    assert lib.osmx_softmax(2, None, 10, fake, 10, 4, 10, ws, 1 << 20, None) == _lib.ERR_INVALID_ARG
    assert lib.osmx_softmax(2, fake, 10, fake, 10, 4, 10, ws, 16, None) == _lib.ERR_INVALID_ARG
    assert lib.osmx_normalizer(fake, 10, 4, 10, -1, fake, fake, ws, 1 << 20, None) == _lib.ERR_INVALID_CHUNK
    # rows == 0 is a no-op
    assert lib.osmx_softmax(2, fake, 10, fake, 10, 0, 10, ws, 1 << 20, None) == _lib.OK


def test_workspace_sizes():
    lib = _lib.load()
    assert lib.osmx_workspace_bytes(2, 4000, 1000, 0) >= 128
    # the unfused pipelines materialise the probability matrix (topk.cpp:33)
    assert lib.osmx_workspace_bytes(6, 4000, 1000, 5) >= 4000 * 1000 * 4
    assert lib.osmx_workspace_bytes(3, 4000, 1000, 5) >= 4000 * 1000 * 4
    # the fused top-K needs no intermediate
    assert lib.osmx_workspace_bytes(5, 4000, 1000, 5) < 1 << 16
    assert lib.osmx_record_bytes(5) % 16 == 0 and lib.osmx_record_bytes(5) >= 16 + 20 + 40


def test_config_knobs_roundtrip():
    for key, val in (("shape", 2), ("split_chunk", 4096), ("topk_threads", 32), ("tma", 2)):
        old = _lib.config_get(key)
        _lib.config_set(key, val)
        assert _lib.config_get(key) == val
        _lib.config_set(key, old)
    with pytest.raises(ValueError):
        _lib.config_set("no_such_knob", 1)


def test_product_path_has_no_oracle_dependency():
    """The product package must not import / link the checker."""
    pkg = ROOT / "paper_1805_02867_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert "from oracle" not in src and "import oracle" not in src, py
    ldd = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "osmx_oracle" not in ldd and "osmx_ref" not in ldd
