"""Compile-time resource guards on the built library (no GPU needed): every
K4 instance keeps its arguments in the parameter bank (a runtime index into
AttnArgs' peer-pointer array once put the whole struct on the local stack,
STACK 16 -> 136 bytes, and cost ~1 us per layer) and no kernel spills."""

import re
import shutil
import subprocess

import pytest

from paper_2602_20732_b200 import _lib


def _resources():
    if shutil.which("cuobjdump") is None or not _lib.LIB_PATH.exists():
        pytest.skip("cuobjdump or the built library missing")
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", str(_lib.LIB_PATH)], check=True,
                         capture_output=True, text=True).stdout
    res = {}
    lines = out.splitlines()
    for i, line in enumerate(lines):
        m = re.search(r"Function (\S+):", line)
        if m and i + 1 < len(lines):
            stats = dict((k, int(v)) for k, v in re.findall(r"(REG|STACK|LOCAL):(\d+)", lines[i + 1]))
            res[m.group(1)] = stats
    assert res, "no kernels found"
    return res


def test_k4_arguments_stay_in_the_parameter_bank():
    res = _resources()
    k4 = {k: v for k, v in res.items() if "sparse_decode_kernel" in k or "sparse_decode_tc_kernel" in k}
    assert k4
    for name, st in k4.items():
        assert st.get("STACK", 0) <= 64, (name, st)


def test_no_local_memory_spills():
    for name, st in _resources().items():
        assert st.get("LOCAL", 0) == 0, (name, st)
