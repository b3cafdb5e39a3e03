"""The C-ABI library loads without a GPU, exports every symbol include/*.h
declares, its struct layouts match the ctypes mirror, and host-side
validation maps onto the pagesel exception classes.  No compute calls."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.errors import ConfigurationError

HEADER = Path(__file__).resolve().parent.parent / "include" / "chess_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(chess_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported(lib):
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    # the ctypes binding covers exactly the declared surface
    assert set(_lib.SIGNATURES) == set(names)


def test_struct_layouts(lib):
    assert lib.chess_abi_version() == _lib.ABI_VERSION
    assert lib.chess_dims_sizeof() == C.sizeof(_lib.ChessDims)
    assert lib.chess_state_sizeof() == C.sizeof(_lib.ChessState)


def _dims(**kw):
    d = _lib.ChessDims()
    vals = dict(batch=2, layers=2, kv_heads=8, q_heads=8, head_dim=64, page_size=16, pages_per_chunk=8,
                chunks_per_grid=8, max_pages=64, window_pages=4, max_ws=64, summary_dtype=0, n_phys=100)
    vals.update(kw)
    for k, v in vals.items():
        setattr(d, k, v)
    d.dim = d.layers * d.kv_heads * d.head_dim if "dim" not in kw else kw["dim"]
    d.ld = d.dim if "ld" not in kw else kw["ld"]
    return d


def test_validate_dims_and_workspace(lib):
    d = _dims()
    assert lib.chess_validate_dims(C.byref(d)) == _lib.OK
    assert lib.chess_workspace_bytes(C.byref(d)) > 0
    for bad in (dict(batch=0), dict(page_size=0), dict(pages_per_chunk=0), dict(window_pages=0),
                dict(q_heads=12), dict(dim=7), dict(ld=1030), dict(n_phys=0), dict(summary_dtype=4),
                dict(summary_dtype=3, ld=1028)):
        d = _dims(**bad)
        rc = lib.chess_validate_dims(C.byref(d))
        assert rc == _lib.ERR_CONFIG, bad
        assert lib.chess_workspace_bytes(C.byref(d)) == 0
        with pytest.raises(ConfigurationError):
            _lib.check(rc, "validate")


def test_tensor_core_summary_dims(lib):
    """summary_dtype 3 (fp16 mirrors scored on tcgen05): 64-element K blocks
    and 8-row groups of children; other fan-outs have no kernel instance."""
    d = _dims(summary_dtype=3)
    assert lib.chess_validate_dims(C.byref(d)) == _lib.OK
    assert lib.chess_workspace_bytes(C.byref(_dims(summary_dtype=3))) > lib.chess_workspace_bytes(C.byref(_dims()))
    d = _dims(summary_dtype=3, pages_per_chunk=4)
    assert lib.chess_validate_dims(C.byref(d)) == _lib.ERR_UNSUPPORTED


def test_status_mapping():
    from paper_2602_20732_b200.errors import EmptyContextError, OutOfPagesError

    with pytest.raises(OutOfPagesError):
        _lib.check(_lib.ERR_OUT_OF_PAGES)
    with pytest.raises(EmptyContextError):
        _lib.check(_lib.ERR_EMPTY_CONTEXT)
    with pytest.raises(ValueError):
        _lib.check(_lib.ERR_SHAPE)
    with pytest.raises(IndexError):
        _lib.check(_lib.ERR_INDEX)
    with pytest.raises(_lib.NativeLibraryError):
        _lib.check(_lib.ERR_CUDA)


def test_host_validation_before_launch(lib):
    # argument errors are reported host-side, before any device work
    assert lib.chess_mean_rows(None, 0, 0, 4, 4, None, None) == _lib.ERR_EMPTY_CONTEXT
    assert lib.chess_page_uncertainty(None, 0, None, None) == _lib.ERR_VALUE
    assert lib.chess_working_set(None, 0, 4, 0, 1, None, None, None, None, None, None) == _lib.ERR_CONFIG
    assert lib.chess_entropy_probs(None, 1, 0, 0, None, None, None) == _lib.ERR_SHAPE
    assert "bad shape" in _lib.last_error()


def test_config_struct_layouts_match_header(tmp_path):
    """Field offsets of the by-pointer config structs, as gcc lays them out
    from include/chess_b200.h, equal the ctypes mirror's."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    structs = {name: getattr(_lib, name) for name in
               ("ChessSelectCfg", "ChessTriggerCfg", "ChessPeerExchange", "ChessPeerOutputs", "ChessDims")}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "chess_b200.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} sizeof %zu\\n", sizeof({name}));')
        for f in cls._fields_:
            lines.append(f'  printf("{name} {f[0]} %zu\\n", offsetof({name}, {f[0]}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(HEADER.parent), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    for line in filter(None, out):
        name, field, value = line.split()
        cls = structs[name]
        want = C.sizeof(cls) if field == "sizeof" else getattr(cls, field).offset
        assert int(value) == want, (name, field, value, want)
