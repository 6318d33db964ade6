"""Input generator: Philox known-answer vectors, shard invariance, recipe ranges."""
import ctypes as C
import os

import numpy as np
import pytest

import synth


@pytest.fixture(scope="module")
def philox_lib(tmp_path_factory):
    src = tmp_path_factory.mktemp("kat") / "kat.c"
    src.write_text('#include "%s"\n' % os.path.join(synth._HERE, "synth_core.h") +
                   "void kat(const unsigned *c, const unsigned *k, unsigned *o){ sy_u4 r = sy_philox(c[0],c[1],c[2],c[3],k[0],k[1]);"
                   " for(int i=0;i<4;++i) o[i]=r.v[i]; }\n")
    so = src.with_suffix(".so")
    assert os.system(f"gcc -O1 -shared -fPIC {src} -o {so}") == 0
    lib = C.CDLL(str(so))
    def run(c, k):
        cc = (C.c_uint * 4)(*c); kk = (C.c_uint * 2)(*k); oo = (C.c_uint * 4)()
        lib.kat(cc, kk, oo)
        return list(oo)
    return run


def test_philox4x32_10_known_answers(philox_lib):
    # Random123 kat_vectors, philox4x32 R=10
    assert philox_lib([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert philox_lib([0xffffffff] * 4, [0xffffffff] * 2) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert philox_lib([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0]) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_deterministic_and_shard_invariant():
    sp, _ = synth.config(2, num_scen=200, rows_pct=20)
    a = synth.generate_host(sp)
    b = synth.generate_host(sp)
    for k in ("n", "r", "d", "t_p", "slo_us"):
        assert np.array_equal(getattr(a, k), getattr(b, k))
    # scenarios [120, 200) drawn as their own shard equal the tail of the full draw
    tail = synth.generate_host(sp.replace(scen_base=120, num_scen=80))
    ref = a.subset(range(120, 200))
    for k in ("scen_dnn_off", "dnn_row_off", "t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax"):
        assert np.array_equal(getattr(tail, k), getattr(ref, k)), k
    R = ref.num_rows
    for k in ("n", "r", "d"):
        assert np.array_equal(getattr(tail, k)[:R], getattr(ref, k)[:R]), k


def test_recipe_ranges():
    sp, pr = synth.config(3, num_scen=300)
    pb = synth.generate_host(sp)
    nd = np.diff(pb.scen_dnn_off)
    assert nd.min() >= 4 and nd.max() <= 16
    assert (pb.slo_us % pr.slot_us == 0).all() and pb.slo_us.min() >= 25000 and pb.slo_us.max() <= 100000
    assert pb.asm_us.min() >= 240 and pb.asm_us.max() <= 1920
    R = pb.num_rows
    r = pb.r[:R]
    assert set(np.unique(r).tolist()) <= {1, 2, 3} and 0.75 < (r == 1).mean() < 0.85
    n = pb.n[:R]
    assert n.min() >= 1 and n.max() <= 4 * 148
    rows = np.diff(pb.dnn_row_off)
    assert rows.min() >= 50 and rows.max() <= 300
    # BERT: 12 identical blocks
    for k in np.flatnonzero(pb.shape == 3)[:5]:
        r0, r1 = pb.dnn_row_off[k], pb.dnn_row_off[k + 1]
        blk = (r1 - r0) // 12
        nn = pb.n[r0:r1].reshape(12, blk)
        assert (nn == nn[0]).all()


def test_paper_mix_config1():
    sp, pr = synth.config(1)
    pb = synth.generate_host(sp)
    assert pb.num_scen == 1 and pb.num_dnn == 4
    assert pb.shape.tolist() == [1, 2, 3, 0]                       # ResNet-50, VGG-19, BERT, MobileNet
    assert pb.slo_us.tolist() == [50000, 100000, 25000, 25000]     # Table 4
    assert pb.asm_us.tolist() == [481] * 4


def test_threads_variant_same_waves():
    sp, _ = synth.config(2, num_scen=50, rows_pct=30)
    a = synth.generate_host(sp)
    b = synth.generate_host(sp.replace(threads=1))
    R = a.num_rows
    th = b.n[:R].astype(np.int64)
    assert ((th + 2047) // 2048 == a.n[:R]).all()
