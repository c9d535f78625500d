"""The C-ABI library loads on a CPU-only host and exports every symbol
include/mhar_b200.h declares; the host-side projector (no GPU) matches the
oracle.  No device compute here."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2104_07097_b200 as mh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "mhar_b200.h")).read()
    return sorted(set(re.findall(r"\b(mhar_[a-z_]+)\s*\(", text)))


def test_header_and_python_symbol_list_agree():
    assert _declared() == sorted(mh.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", mh.library_path()], check=True,
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(mhar_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    L = mh.lib()
    for s in _declared():
        assert hasattr(L, s)


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", mh.library_path()], check=True,
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", mh.library_path()], check=True,
                          capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass      # fp64 tensor-core MMA
    assert "UBLKCP" in sass          # TMA bulk copies feeding the chord kernel


def test_version_and_last_error():
    assert b"sm_100a" in mh.lib().mhar_version()
    with pytest.raises(mh.MharError) as e:
        mh.compute_projection(np.eye(3))
    assert e.value.code == mh.ErrorCode.rank_deficient_eq
    assert "RANK_DEFICIENT_EQ" in str(e.value)


def test_host_projection_matches_oracle(orc):
    rng = np.random.default_rng(5)
    for me, n in [(1, 3), (1, 100), (5, 12), (20, 60), (100, 1000)]:
        AE = rng.standard_normal((me, n))
        op = mh.compute_projection(AE)
        st, P, G = orc.compute_projection(AE)
        assert st == 0
        np.testing.assert_allclose(op.p, P, rtol=0, atol=1e-12)
        np.testing.assert_allclose(op.gram_inverse, G, rtol=1e-10, atol=1e-14)
        assert np.abs(op.p @ op.p - op.p).max() <= 1e-9
        assert np.abs(AE @ op.p).max() <= 1e-9 * max(1.0, np.abs(AE).max())
    # the simplex projector is exact (acceptance_main.cpp:122-125)
    op = mh.compute_projection(np.ones((1, 4)))
    want = np.full((4, 4), -0.25)
    np.fill_diagonal(want, 0.75)
    assert np.array_equal(op.p, want)
    with pytest.raises(mh.MharError) as e:
        mh.compute_projection(np.array([[1, 1, 0, 0], [2, 2, 0, 0.0]]))
    assert e.value.code == mh.ErrorCode.rank_deficient_eq


def test_resolve_defaults_and_validation():
    # proj/tests/test_sampler.cpp:29-76
    cube = mh.make_hypercube(5)
    rc = mh.resolve(mh.SamplerConfig(), cube)
    assert (rc.z, rc.phi, rc.burn_in, rc.reproject_every) == (11, 125, 125, 125)
    rs = mh.resolve(mh.SamplerConfig(), mh.make_simplex(4))
    assert (rs.z, rs.phi) == (5, 27)
    re_ = mh.resolve(mh.SamplerConfig(z=7, phi=9, burn_in=0, reproject_every=0), cube)
    assert (re_.z, re_.phi, re_.burn_in, re_.reproject_every) == (7, 9, 0, 0)
    for bad in [mh.SamplerConfig(z=-2), mh.SamplerConfig(t_target=0),
                mh.SamplerConfig(eps_dir=0.0), mh.SamplerConfig(eps_feas=-1.0)]:
        with pytest.raises(mh.MharError) as e:
            mh.resolve(bad, mh.make_hypercube(3))
        assert e.value.code == mh.ErrorCode.invalid_argument


def test_layout_index_maps_are_bijections():
    # The packed operand layouts (csrc/common.cuh) restated in numpy: every
    # (row|walk, k) lands on a distinct slot of its tile.
    BM, BK, BC = 128, 16, 64

    def a_index(r, k, KT):
        mt, rr = divmod(r, BM)
        rg, rin = divmod(rr, 8)
        kt, kk = divmod(k, BK)
        k8, kin = divmod(kk, 8)
        e, kq = divmod(kin, 4)
        lane = rin * 4 + kq
        return ((((mt * KT + kt) * 2 + k8) * 16 + rg) * 32 + lane) * 2 + e

    def b_index(c, k, KT):
        ct, cc = divmod(c, BC)
        cg, cin = divmod(cc, 8)
        kt, kk = divmod(k, BK)
        k8, kin = divmod(kk, 8)
        e, kq = divmod(kin, 4)
        lane = cin * 4 + kq
        return ((((ct * KT + kt) * 2 + k8) * 8 + cg) * 32 + lane) * 2 + e

    KT = 3
    r, k = np.meshgrid(np.arange(2 * BM), np.arange(KT * BK), indexing="ij")
    ai = a_index(r, k, KT).ravel()
    assert len(np.unique(ai)) == ai.size and ai.min() == 0 and ai.max() == ai.size - 1
    c, k = np.meshgrid(np.arange(2 * BC), np.arange(KT * BK), indexing="ij")
    bi = b_index(c, k, KT).ravel()
    assert len(np.unique(bi)) == bi.size and bi.min() == 0 and bi.max() == bi.size - 1
