"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
public header declares (host-only checks; no device work)."""

import os
import re
import subprocess

from conftest import ROOT


def _declared():
    with open(os.path.join(ROOT, "include", "citywalk_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|long long)\s+(cw_\w+)\s*\(", text, re.M)))


def test_header_declares_the_exports():
    from paper_2505_00690_b200 import _lib
    assert sorted(_lib.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol():
    from paper_2505_00690_b200 import _lib
    _lib.build()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for s in _declared():
        assert s in syms, s


def test_library_loads_and_abi_structs_agree():
    from paper_2505_00690_b200 import _lib
    L = _lib.lib()   # raises on an ABI size mismatch
    assert L.cw_scene_seed_scratch_bytes(10) > 0
    assert L.cw_crowd_step_smem_bytes(32, 128) > 0


def test_sm100a_code_in_library():
    from paper_2505_00690_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
