"""The C-ABI library: loads without a GPU, exports every symbol the headers
declare, validates like lp2d::solve_batch (batch.hpp:305-320), and fails
loudly instead of falling back to the CPU. CPU only."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, cuda_available


def declared_functions():
    names = []
    for h in ("lp2d_b200.h", "lp2d_b200_gen.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"^\s*(?:[\w*]+\s+)+\**(lp2d\w+)\s*\(", src, re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol(P):
    L = P.lp2d.N.lib()
    decl = declared_functions()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(P.lp2d.N.EXPORTS)
    assert b"sm_100a" in L.lp2dgpu_version()


def test_pack_offsets_contract(P):
    m = np.array([0, 1, 7, 8, 9, 1024, 3], np.int32)
    off = P.lp2d.pack_offsets(m)
    assert off[0] == 0 and np.all(off % 8 == 0)
    assert np.all(np.diff(off) >= (m + 7) // 8 * 8)


def test_partition_balances_work(P):
    from paper_1902_04995_b200 import sharding

    m = np.array([8] * 90 + [8192] * 10, np.int32)
    cut = sharding.partition(m, 4)
    assert cut[0] == 0 and cut[-1] == 100 and np.all(np.diff(cut) >= 0)
    w = [(m[cut[g]:cut[g + 1]] + 4).sum() for g in range(4)]
    assert max(w) <= (m + 4).sum() / 4 + 8192 + 4


def _batch(P):
    return P.gen_mixed([10], 2, 1)


def test_solve_batch_validates_like_the_reference(P):
    # test_batch.cpp:169-184
    with pytest.raises(ValueError):
        P.solve_batch(P.Batch())
    b = _batch(P)
    b.permutations.pop()
    with pytest.raises(ValueError):
        P.solve_batch(b)
    c = _batch(P)
    c.permutations[1] = P.Permutation(c.permutations[1].order[:-1])
    with pytest.raises(ValueError):
        P.solve_batch(c)
    with pytest.raises(ValueError):
        P.solve_batch(_batch(P), P.BlockConfig(block_width=0))


def test_c_abi_error_codes(P):
    import ctypes as C

    N = P.lp2d.N
    L = N.lib()
    o = N.Opts()
    L.lp2dgpu_default_opts(C.byref(o))
    s = N.BatchSoA()
    r = N.Out()
    assert L.lp2dgpu_solve_f32(C.byref(s), C.byref(o), C.byref(r)) == N.ERR_EMPTY_BATCH
    s.n = 1
    o.block_width = 0
    assert L.lp2dgpu_solve_f32(C.byref(s), C.byref(o), C.byref(r)) == N.ERR_BLOCK_WIDTH
    o.block_width = 512
    s.perm_bits = 7
    assert L.lp2dgpu_solve_f64(C.byref(s), C.byref(o), C.byref(r)) == N.ERR_ARG
    assert "perm_bits" in N.last_error()


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(P):
    pb = P.PackedBatch.generate(np.full(4, 16, np.int32), 3)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.solve_packed(pb)


def test_perm_seed_api_validation(P):
    pb = P.PackedBatch.generate(np.array([5, 6], np.int32), 1)
    noperm = P.PackedBatch(pb.m, pb.offset, pb.ax, pb.ay, pb.b, None, pb.c, pb.M)
    with pytest.raises(ValueError):
        P.solve_packed(noperm)  # neither perm nor perm_seed
    f = {n for n, _ in P.lp2d.N.BatchSoA._fields_}
    assert {"perm_from_seed", "perm_mul", "perm_add", "perm_seed", "perm_first"} <= f
