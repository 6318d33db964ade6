"""The C-ABI library loads and exports every symbol include/dstack.h declares (CPU; no compute calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:dstack|synth)_\w+)\s*\(", src)))


def test_libdstack_exports_every_declared_symbol():
    lib = C.CDLL(os.path.join(ROOT, "paper_2304_13541_b200", "libdstack.so"))
    names = declared("dstack.h")
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    from paper_2304_13541_b200 import dstack
    assert set(dstack.EXPORTS) == set(names)


def test_synth_libs_export_declared_symbols():
    names = declared("dstack_synth.h")
    host = C.CDLL(os.path.join(ROOT, "synth", "libdstack_synth_host.so"))
    dev = C.CDLL(os.path.join(ROOT, "synth", "libdstack_synth_dev.so"))
    for n in names:
        assert hasattr(host if n.startswith("synth_host") else dev, n), n


def test_host_side_argument_checks():
    from paper_2304_13541_b200 import dstack as ds
    lib = ds.lib()
    assert lib.dstack_version() == 1
    pb = ds.CProblem(0, 0, 0, *([None] * 11))
    good = ds.CParams(100, 148, 100, 1, 0, 0, 0, 1, 64, 0)
    assert lib.dstack_workspace_size(C.byref(pb), C.byref(good)) > 0
    for bad in (ds.CParams(0, 148, 100, 1, 0, 0, 0, 1, 64, 0), ds.CParams(100, 300, 100, 1, 0, 0, 0, 1, 64, 0),
                ds.CParams(100, 148, 100, 3, 0, 0, 0, 1, 64, 0), ds.CParams(100, 148, 100, 1, 0, 0, 0, 2, 1, 0),
                ds.CParams(100, 148, 100, 1, 0, 0, 0, 1, 65, 0), ds.CParams(100, 148, 0, 1, 0, 0, 0, 1, 64, 0),
                ds.CParams(100, 148, 100, 1, 0, 0, 0, 1, 64, 4), ds.CParams(100, 148, 100, 1, 0, 0, 0, 1, 64, 2, -1)):
        assert lib.dstack_batch_opt(C.byref(pb), C.byref(bad), None, None, None, None, None, 0, None) == ds.DSTACK_EINVAL
    # missing outputs for a non-empty problem
    pb1 = ds.CProblem(1, 1, 1, *([8] * 11))
    assert lib.dstack_batch_opt(C.byref(pb1), C.byref(good), None, None, None, None, None, 0, None) == ds.DSTACK_EINVAL
    assert lib.dstack_status_str(ds.DSTACK_EWORKSPACE).startswith(b"EWORKSPACE")
    # F1 is rejected where it is not implemented (dstack.h)
    bk = ds.CParams(100, 148, 100, 1, 0, 0, 0, 1, 64, ds.FLAG_BELOW_KNEE, 100)
    assert lib.dstack_workspace_size(C.byref(pb), C.byref(bk)) > 0
    assert lib.dstack_compare(C.byref(pb), C.byref(bk), None, None, None, None, None, None, None, 0,
                              None) == ds.DSTACK_EINVAL
    assert lib.dstack_cluster(C.byref(pb), C.byref(bk), 4, None, None, None, None, None, 0, None) == ds.DSTACK_EINVAL
    assert lib.dstack_cluster(C.byref(pb), C.byref(good), 0, None, None, None, None, None, 0, None) == ds.DSTACK_EINVAL
    assert lib.dstack_cluster(C.byref(pb), C.byref(good), 33, None, None, None, None, None, 0, None) == ds.DSTACK_EINVAL


def test_struct_layouts_match_header():
    from paper_2304_13541_b200 import dstack as ds
    # dstack_agg_t: 5 doubles + 4 + 5 + 5 + 3 + 65 + 256 + 1 u64
    assert C.sizeof(ds.CAgg) == 8 * (5 + 4 + 5 + 5 + 3 + 65 + 256 + 1)
    assert C.sizeof(ds.CProblem) == 4 + 4 + 8 + 11 * 8
    assert C.sizeof(ds.CParams) == 11 * 4
    assert C.sizeof(ds.COut) == 18 * 8


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is not None and False, reason="")
def test_product_does_not_import_oracle():
    # the product package and its sources never reference oracle/
    pkg = os.path.join(ROOT, "paper_2304_13541_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f
