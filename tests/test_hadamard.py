"""The Walsh-Hadamard oracle (oracle/hadamard.py) pinned against a library routine, SPEC.md's
worked examples and closed forms (CPU), and the library's paro_fwht against it (GPU).
PAPER.md:200-209 (fig:kernel-speedup's comparison transform)."""
import numpy as np
import pytest

from oracle import hadamard as H


def test_matches_scipy_hadamard():
    scipy_linalg = pytest.importorskip("scipy.linalg")
    for n in (1, 2, 4, 64, 256):
        assert np.array_equal(H.hadamard_matrix(n), scipy_linalg.hadamard(n))


def test_spec_examples():
    assert np.array_equal(H.fwht(np.array([[1.0, 0, 0, 0]])), [[1, 1, 1, 1]])
    v = np.random.default_rng(0).normal(size=(3, 64))
    assert np.allclose(H.fwht(H.fwht(v)), 64 * v, atol=1e-12)                   # SPEC.md:342 involution


def test_closed_form_and_orthogonality():
    n = 32
    M = H.hadamard_matrix(n)
    for i in range(n):
        for j in range(n):
            assert M[i, j] == (-1) ** bin(i & j).count("1")
    assert np.array_equal(M @ M.T, n * np.eye(n))
    # randomised orthogonal variant preserves the norm
    rng = np.random.default_rng(1)
    x = rng.normal(size=(2, 1024))
    s = rng.choice([-1.0, 1.0], size=1024)
    y = H.fwht(x, s, 1.0 / np.sqrt(1024))
    assert np.allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [256, 512, 1024, 2048, 4096, 8192, 16384])
@pytest.mark.parametrize("T", [1, 3, 37])
def test_paro_fwht_parity(n, T):
    torch = pytest.importorskip("torch")
    import paper_2511_10645_b200 as paro
    import oracle as O
    rng = np.random.default_rng(n + T)
    x = rng.normal(size=(T, n)).astype(np.float16)
    s = rng.choice([-1.0, 1.0], size=n).astype(np.float32)
    scale = 1.0 / np.sqrt(n)
    y = paro.paro_fwht(torch.from_numpy(x).cuda(), torch.from_numpy(s).cuda(), scale)
    torch.cuda.synchronize()
    ref = H.fwht(x.astype(np.float64), s, scale)
    assert O.normwise_error(y.float().cpu().numpy(), ref) <= 2e-3
    # unnormalised, no signs, bf16 input
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    y2 = paro.paro_fwht(xb, None, 1.0 / 64)
    torch.cuda.synchronize()
    ref2 = H.fwht(xb.float().cpu().numpy().astype(np.float64), None, 1.0 / 64)
    assert O.normwise_error(y2.float().cpu().numpy(), ref2) <= 2e-3


@pytest.mark.gpu
def test_paro_fwht_errors():
    torch = pytest.importorskip("torch")
    import paper_2511_10645_b200 as paro
    x = torch.zeros((2, 384), dtype=torch.float16, device="cuda")
    with pytest.raises(paro.ParoError) as e:
        paro.paro_fwht(x)
    assert e.value.kind == "unsupported"
