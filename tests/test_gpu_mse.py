"""GPU MSE scale search vs the reference's own outputs.

Fixtures: ``tests/golden/mse_fixtures.npz`` from ``tests/golden/make_mse.py``, which runs the
unmodified reference ``quantize(X, spec, ScalePolicy(mode=MSE), transform)``
(pkg/src/microfp/quantizers.py:330-347; search ``optimize_group_scales`` :263-327).
Bar: codes and scale codes >= 99.99% identical (bit-exact expected), tensor scale equal,
metrics within 1e-6 relative.
"""

import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2509_23202_b200 as P

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
MSE = np.load(os.path.join(HERE, "golden", "mse_fixtures.npz"))
CASES = sorted({k[: -len("_codes")] for k in MSE.files if k.endswith("_codes")})


def _spec(key):
    return P.FormatSpec.mxfp4() if key.startswith("mx") else P.FormatSpec.nvfp4()


def _k(key):
    return int(key.split("_")[1][1:])


@pytest.mark.parametrize("key", CASES)
def test_mse_matches_reference(key):
    X = torch.from_numpy(MSE[key + "_x"]).cuda().bfloat16()
    pol = P.ScalePolicy(mode=P.ScaleMode.MSE, e8m0_four_thirds=not key.endswith("no43"))
    k = _k(key)
    r = P.quantize(X, _spec(key), policy=pol, transform=P.TransformSpec.hadamard(k) if k else None)
    codes = r.codes.cpu().numpy()
    scales = r.scale_codes().cpu().numpy()
    ref_c, ref_s = MSE[key + "_codes"], MSE[key + "_scales"]
    assert r.tensor_scale == float(MSE[key + "_ts"])
    assert (scales == ref_s).mean() >= 0.9999, (scales != ref_s).sum()
    assert (codes == ref_c).mean() >= 0.9999, (codes != ref_c).sum()
    assert np.array_equal(scales, ref_s) and np.array_equal(codes, ref_c)
    np.testing.assert_allclose([r.mse_rel, r.mse_top_rel], MSE[key + "_mse"], rtol=1e-6)


def test_mse_never_worse_than_absmax():
    """quantizers.py:268-270: the search starts from the absmax assignment and only improves."""
    rng = np.random.default_rng(4)
    X = torch.from_numpy(O.bf16_round(rng.laplace(size=(128, 2048)))).cuda().bfloat16()
    for spec, k in ((P.FormatSpec.nvfp4(), 16), (P.FormatSpec.mxfp4(), 32)):
        tr = P.TransformSpec.hadamard(k)
        rtn = P.quantize_rtn(X, spec, transform=tr)
        mse = P.quantize(X, spec, policy=P.ScalePolicy(mode=P.ScaleMode.MSE), transform=tr)
        assert mse.mse_rel <= rtn.mse_rel


def test_mse_underflow_raises_like_reference():
    assert bool(MSE["nv_underflow_raises"])
    X = torch.from_numpy(MSE["nv_underflow_x"]).cuda()
    with pytest.raises(P.DataError):
        P.quantize(X, P.FormatSpec.nvfp4(), policy=P.ScalePolicy(mode=P.ScaleMode.MSE))


def test_quantize_rtn_ignores_policy_mode():
    """The reference's quantize_rtn never looks at policy.mode (quantizers.py:247-255)."""
    rng = np.random.default_rng(5)
    X = torch.from_numpy(O.bf16_round(rng.standard_normal((64, 1024)))).cuda().bfloat16()
    a = P.quantize_rtn(X, P.FormatSpec.nvfp4(), policy=P.ScalePolicy(mode=P.ScaleMode.MSE))
    b = P.quantize_rtn(X, P.FormatSpec.nvfp4())
    assert torch.equal(a.codes, b.codes) and torch.equal(a.sf, b.sf)


def test_mse_weight_feeds_the_linear():
    """An MSE-quantized weight goes through prepare_weight and the GEMM like any other."""
    rng = np.random.default_rng(6)
    W = O.bf16_round(rng.standard_normal((256, 1024)) / 32)
    X = O.bf16_round(rng.standard_normal((64, 1024)))
    tr = P.TransformSpec.hadamard(16)
    wq = P.quantize(torch.from_numpy(W).cuda(), P.FormatSpec.nvfp4(), policy=P.ScalePolicy(mode=P.ScaleMode.MSE),
                    transform=tr)
    w = P.prepare_weight(wq)
    y = P.quantized_linear(torch.from_numpy(X).cuda().bfloat16(), w, out_dtype=torch.float32).cpu().numpy()
    t = wq.to_mfp()
    ec = O.unpack_nibbles(np.asarray(t.codes), t.rows * t.cols).reshape(t.rows, t.cols)
    Wo = O.OracleQuant("nvfp4", t.rows, t.cols, 16, 16, ec, np.asarray(t.scale_codes).reshape(t.rows, -1),
                       t.tensor_scale, 0.0, 0.0)
    ref = O.linear_reference(O.quantize_rtn(X, "nvfp4", hadamard=16), Wo)
    assert float(np.linalg.norm(y - ref) / np.linalg.norm(ref)) <= 1e-5


@pytest.mark.parametrize("n", [1, 7, 8, 100, 128, 129, 2048, 16384, 16385, 100003, 1 << 20])
def test_gpu_pairwise_sum_is_numpy_sum(n):
    """The MSE driver's device sums reproduce np.sum bit for bit (numpy's pairwise recursion)."""
    from paper_2509_23202_b200.quantize import _NpSum
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) ** 2 * 10.0 ** rng.integers(-8, 8, n)
    t = torch.from_numpy(a).cuda()
    assert _NpSum.whole(n, "cuda").total(t) == float(np.sum(a))
    ch = _NpSum.chunks(n, 2048, "cuda").segment_sums(t)
    assert all(float(c) == float(np.sum(a[i * 2048:(i + 1) * 2048])) for i, c in enumerate(ch))
