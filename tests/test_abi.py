"""CPU-only checks of the C ABI boundary: libseqcdc.so builds for sm_100a,
loads without a GPU, exports every function include/*.h declares, and its
host-side parameter logic behaves as documented.  No compute calls."""
import glob
import os
import re

import pytest

import paper_2505_21194_b200 as sc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(seqcdc_[a-z_0-9]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = sc.lib()
    declared = _declared_functions()
    assert len(declared) >= 10
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(sc.EXPORTS) <= declared | set(sc.EXPORTS)
    for n in sc.EXPORTS:
        assert n in declared, f"{n} exported by the binding but not declared in include/"


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {sc._build.LIB} 2>/dev/null").read()
    assert "sm_100a" in out


def test_validate_params():
    assert sc.validate(sc.SeqParams())
    bad = [
        sc.SeqParams(mode=2), sc.SeqParams(seq_length=1), sc.SeqParams(seq_length=17, min_size=4096),
        sc.SeqParams(skip_trigger=0), sc.SeqParams(min_size=4), sc.SeqParams(min_size=100, max_size=99),
    ]
    for p in bad:
        assert not sc.validate(p), p
    assert sc.validate(sc.SeqParams(seq_length=16, min_size=16, max_size=16))
    assert sc.validate(sc.SeqParams(seq_length=2, skip_trigger=1, skip_size=0, min_size=2, max_size=2))
    # flags: signed and comparisons readings; the latter needs L+1 <= 16 bytes per run
    assert sc.validate(sc.SeqParams(flags=sc.FLAG_SIGNED | sc.FLAG_PAIRS))
    assert sc.validate(sc.SeqParams(seq_length=15, min_size=16, max_size=16, flags=sc.FLAG_PAIRS))
    assert not sc.validate(sc.SeqParams(seq_length=16, min_size=16, max_size=16, flags=sc.FLAG_PAIRS))
    assert not sc.validate(sc.SeqParams(flags=4))


def test_default_params_table1():
    """Table I with min = avg/2, max = 2 avg."""
    assert sc.SeqParams.table1(4) == sc.SeqParams(0, 5, 55, 256, 2048, 8192)
    assert sc.SeqParams.table1(8, 1) == sc.SeqParams(1, 5, 50, 256, 4096, 16384)
    assert sc.SeqParams.table1(16) == sc.SeqParams(0, 5, 50, 512, 8192, 32768)
    with pytest.raises(sc.SeqCDCError):
        sc.SeqParams.table1(32)


def test_max_cuts_bounds():
    p = sc.SeqParams.table1(8)
    assert sc.max_cuts(0, p) == 0
    assert sc.max_cuts(1, p) == 1
    assert sc.max_cuts(4096, p) == 1
    assert sc.max_cuts(4097, p) == 2
    assert sc.max_cuts_batch(10 * 4096, 3, p) == 13


def test_workspace_size_is_host_only():
    p = sc.SeqParams.table1(8)
    ws = sc.workspace_size(1 << 30, 1, p)
    assert 0 < ws < (1 << 30)
