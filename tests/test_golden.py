"""Golden vectors made by the UNMODIFIED reference (tests/golden/make_golden.py):
the oracle must reproduce them bit for bit (CPU), and libarfx must reproduce the
integer decisions bit for bit and the f32 outputs within tolerance (GPU)."""
import hashlib
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_golden import OUT, compute, golden_inputs  # noqa: E402

from paper_2212_10550_b200 import arf  # noqa: E402


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(OUT))


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind in "US":
        return a == b
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                                                 np.ascontiguousarray(b).view(np.uint8))


def test_oracle_reproduces_golden(oracle, golden):
    out = compute(oracle)
    assert set(out) == set(golden)
    bad = [k for k in golden if not _eq(out[k], golden[k])]
    assert not bad, f"oracle differs from the reference's golden vectors in {bad}"


@pytest.mark.gpu
def test_gpu_reproduces_golden(gpu, golden):
    I = golden_inputs()
    dm = arf.build_model(I["sk"], I["g"], I["m"], I["skin_res"], I["seed"])
    gp, mp, sw = dm.params()
    assert hashlib.sha256(gp.tobytes()).hexdigest() == str(golden["grid_sha"])
    assert hashlib.sha256(sw.tobytes()).hexdigest() == str(golden["skin_sha"])
    assert np.array_equal(mp.view(np.uint32), golden["mlp"].view(np.uint32))
    lo, hi = golden["boxes"][0], golden["boxes"][1]
    nlo, nhi = golden["boxes"][2], golden["boxes"][3]
    assert np.array_equal(dm.skinning_weights(lo + (hi - lo) * I["skin_unit"]).view(np.uint64),
                          golden["skin_w"].view(np.uint64))
    pts = lo + (hi - lo) * I["unit"]
    assert np.array_equal(dm.encode(pts).view(np.uint32), golden["feats"].view(np.uint32))
    d, c = dm.field_query(pts)
    np.testing.assert_allclose(d, golden["dens"], rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(c, golden["col"], rtol=2e-6, atol=1e-7)
    P = I["pose"]
    cnt, roots, res = dm.inverse_lbs(P, golden["root_pts"], arf.rigid(), 3.0)
    assert np.array_equal(cnt, golden["root_cnt"])
    assert np.array_equal(roots.view(np.uint64), golden["roots"].view(np.uint64))
    q = nlo + (nhi - nlo) * I["norm_unit"]
    pd, pc, px, ph = dm.posed_query(P, q)
    assert np.array_equal(ph, golden["pq_has"].astype(bool))
    occ = arf.build_model_inference_grid(dm, P, I["occ"])
    v, m = occ.download()
    assert np.array_equal(m, golden["occ_mask"])
    np.testing.assert_allclose(v, golden["occ_values"], rtol=2e-6, atol=1e-7)
    img = arf.render_model(dm, P, I["cam"], occ, I["opt"])
    np.testing.assert_allclose(img.rgb, golden["rgb"], rtol=1e-3, atol=1e-5)
    np.testing.assert_allclose(img.alpha, golden["alpha"], rtol=1e-3, atol=1e-5)
    tr = arf.render_trace(dm)
    order = np.lexsort((tr.index, tr.ray))
    assert np.array_equal(tr.ray[order], golden["trace_s_ray"])
    assert np.array_equal(tr.index[order], golden["trace_s_index"])
    assert np.array_equal(tr.delta[order].view(np.uint64), golden["trace_s_delta"].view(np.uint64))
