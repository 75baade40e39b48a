"""Device priors from observations (serial.py:39-50), bit-identical to the reference's numpy.

CPU: the C restatement of numpy's AVX512_SKX exp (oracle/npexp.c) equals np.exp on this
host.  GPU: the device exp and prior kernels equal the restatement bit for bit over the
whole argument range (independent of the host), and decoding observations with device
priors gives exactly the outputs of decoding the host's numpy priors."""

import numpy as np
import pytest

import oracle
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch
from paper_1609_01567_b200 import decoder as decoder_mod


def _host_has_svml_exp() -> bool:
    """numpy >= 2 dispatches float64 exp to SVML on AVX512_SKX hosts."""
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as feats
    except ImportError:  # pragma: no cover
        return False
    return bool(feats.get("AVX512_SKX")) and int(np.__version__.split(".")[0]) >= 2


def _args(seed=0):
    rng = np.random.default_rng(seed)
    fh = float.fromhex
    edges = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-300, 5e-324, 2.0 ** -54, -(2.0 ** -54),
                      fh("0x1.62e42fefa39efp+9"), np.nextafter(fh("0x1.62e42fefa39efp+9"), 1e9),
                      fh("0x1.61da04cbafe44p+9"), -fh("0x1.61da04cbafe44p+9"),
                      np.nextafter(fh("0x1.61da04cbafe44p+9"), 0), fh("-0x1.74910d52d3051p+9"),
                      np.nextafter(fh("-0x1.74910d52d3051p+9"), -1e9), fh("-0x1.6232bdd7abcd2p+9"),
                      np.nextafter(fh("-0x1.6232bdd7abcd2p+9"), 0), -1074 * np.log(2.0), -1080 * np.log(2.0)])
    return np.concatenate([rng.uniform(-40, 40, 400_000), rng.uniform(-750, 715, 200_000),
                           rng.uniform(-746, -705, 100_000), rng.uniform(705, 710, 50_000),
                           rng.normal(0, 1e-12, 10_000), edges,
                           rng.integers(0, 2 ** 64, 100_000, dtype=np.uint64).view(np.float64)])


def _same(a, b):
    return (a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))


# ---- CPU -------------------------------------------------------------------------

def test_oracle_exp_matches_host_numpy():
    if not _host_has_svml_exp():
        pytest.skip("this host's numpy does not run the SVML exp (no AVX512_SKX)")
    x = _args(1)
    with np.errstate(all="ignore"):
        want = np.exp(x)
    assert _same(oracle.npexp(x), want).all()


def test_oracle_prior_matches_reference_expression():
    if not _host_has_svml_exp():
        pytest.skip("this host's numpy does not run the SVML exp (no AVX512_SKX)")
    rng = np.random.default_rng(2)
    for s2 in (0.05, 0.3, 0.6309573444801932, 1.0, 2.5, 1e3):
        y = rng.normal(-1.0, np.sqrt(s2), 50_000) * rng.choice([1.0, -1.0, 40.0], 50_000)
        assert _same(oracle.priors_awgn_svml(y, s2), oracle.priors_awgn(y, s2)).all(), s2


# ---- GPU -------------------------------------------------------------------------

@pytest.mark.gpu
def test_device_exp_matches_restatement(cuda):
    import torch

    from paper_1609_01567_b200 import _native

    x = _args(3)
    xd = torch.from_numpy(x).to(cuda)
    out = torch.empty_like(xd)
    _native.check(_native.lib().ldpc_npexp(xd.data_ptr(), x.size, out.data_ptr(), None), "npexp")
    torch.cuda.synchronize()
    got, want = out.cpu().numpy(), oracle.npexp(x)
    bad = np.nonzero(~_same(got, want))[0]
    assert bad.size == 0, [(x[i], got[i], want[i]) for i in bad[:5]]


@pytest.mark.gpu
def test_device_priors_match_restatement(cuda):
    import torch

    from paper_1609_01567_b200 import _native

    rng = np.random.default_rng(4)
    B, n = 7, 5000
    s2 = rng.uniform(0.05, 3.0, B)
    s2[0] = 1e-3  # huge |x|: rare path and saturation
    Y = rng.normal(-1.0, 1.0, (B, n)) * rng.choice([1.0, 30.0], (B, n))
    yd, sd = torch.from_numpy(Y).to(cuda), torch.from_numpy(s2).to(cuda)
    pd = torch.empty_like(yd)
    _native.check(_native.lib().ldpc_priors_awgn(yd.data_ptr(), sd.data_ptr(), B, n, pd.data_ptr(), None), "priors")
    torch.cuda.synchronize()
    got = pd.cpu().numpy()
    for b in range(B):
        assert _same(got[b], oracle.priors_awgn_svml(Y[b], s2[b])).all(), b


@pytest.mark.gpu
def test_probe_agrees_with_host(cuda):
    exact = decoder_mod.device_priors_exact(0)
    if _host_has_svml_exp():
        assert exact
    x = decoder_mod._exp_probe_inputs()
    with np.errstate(all="ignore"):
        host = np.exp(x)
    assert exact == bool(_same(oracle.npexp(x), host).all())


def _observations(code, B, ebno, seed):
    H = configs.code(code)
    s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
    rng = np.random.default_rng(seed)
    return H, -1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2


def _assert_same(a, b):
    assert np.array_equal(a.est_bits, b.est_bits)
    assert np.array_equal(a.success, b.success)
    assert np.array_equal(a.iterations, b.iterations)
    assert np.array_equal(a.syn_bits, b.syn_bits)


@pytest.mark.gpu
@pytest.mark.parametrize("code,B,ebno,schedule", [("C1", 37, 1.5, "auto"), ("C1", 5, 2.0, "onchip"),
                                                  ("C2", 70, 1.0, "stream"), ("C4", 9, 3.0, "auto")])
def test_decode_observations_equals_host_priors(cuda, monkeypatch, code, B, ebno, schedule):
    if not decoder_mod.device_priors_exact(0):
        pytest.skip("host numpy exp differs from the device prior (host priors are used instead)")
    H, Y, s2 = _observations(code, B, ebno, 11)
    sig = np.linspace(0.8, 1.2, B) * s2  # per-frame noise variances
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        dev = dec.decode_batch(Y, sig, 12, schedule=schedule)
        host = dec.decode_priors(priors_awgn_batch(Y, sig), 12, schedule=schedule)
        _assert_same(dev, host)
        monkeypatch.setenv("LDPC_DEVICE_PRIORS", "0")  # forced host-prior path of decode_batch
        _assert_same(dec.decode_batch(Y, sig, 12, schedule=schedule), host)


@pytest.mark.gpu
def test_decode_observations_streaming_and_chunked(cuda):
    if not decoder_mod.device_priors_exact(0):
        pytest.skip("host numpy exp differs from the device prior")
    H, Y, s2 = _observations("C2", 150, 1.25, 12)
    T = CodeTables.from_matrix(H)
    with ParallelDecoder(T, max_batch=64) as dec:
        ref = dec.decode_priors(priors_awgn_batch(Y, s2), 10)
        _assert_same(dec.decode_batch(Y, s2, 10), ref)  # B > max_batch: chunks through the slots
        jobs = [dec.decode_batch_async(Y[c:c + 64], s2, 10) for c in (0, 64)]
        for c, job in zip((0, 64), jobs):
            got = job.wait()
            assert np.array_equal(got.est_bits, ref.est_bits[c:c + 64])
            assert np.array_equal(got.iterations, ref.iterations[c:c + 64])


@pytest.mark.gpu
def test_single_frame_decode_uses_device_priors(cuda):
    H, Y, s2 = _observations("C1", 3, 1.0, 13)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=1) as dec:
        for y in Y:
            got = dec.decode(y, s2, 20)
            ref = dec.decode_priors(oracle.priors_awgn(y, s2).reshape(1, -1), 20)[0]
            assert np.array_equal(got.estimate, ref.estimate)
            assert got.success == ref.success and got.iterations_used == ref.iterations_used


@pytest.mark.gpu
def test_device_api_observations(cuda):
    import torch

    H, Y, s2 = _observations("C2", 40, 1.5, 14)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=40) as dec:
        sig = torch.full((40,), s2, dtype=torch.float64, device=cuda)
        est, ok, its, syn = dec.decode_device_awgn(torch.from_numpy(Y).to(cuda), sig, 10)
        P = torch.from_numpy(oracle.priors_awgn_svml(Y.ravel(), s2).reshape(Y.shape)).to(cuda)
        est2, ok2, its2, syn2 = dec.decode_device(P, 10)
        torch.cuda.synchronize()
        for a, b in ((est, est2), (ok, ok2), (its, its2), (syn, syn2)):
            assert torch.equal(a, b)


@pytest.mark.gpu
def test_decode_observations_extreme_values(cuda):
    """Saturated priors (p exactly 0 or 1, exp overflow), the rare exp path and subnormal exps."""
    if not decoder_mod.device_priors_exact(0):
        pytest.skip("host numpy exp differs from the device prior")
    H, Y, s2 = _observations("C1", 24, 2.0, 15)
    rng = np.random.default_rng(16)
    mask = rng.random(Y.shape) < 0.02
    Y[mask] = rng.choice([-400.0, -360.0, -354.2, 354.0, 360.0, 1e5, -1e5], mask.sum())
    sig = np.full(24, s2)
    sig[:4] = [1e-3, 0.5, 1.0, 2.0]
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=24) as dec:
        for schedule in ("stream", "onchip"):
            dev = dec.decode_batch(Y, sig, 15, schedule=schedule)
            host = dec.decode_priors(priors_awgn_batch(Y, sig), 15, schedule=schedule)
            _assert_same(dev, host)


@pytest.mark.gpu
def test_decode_observations_nonfinite(cuda):
    """NaN / inf observations: the device prior propagates them exactly like numpy's."""
    if not decoder_mod.device_priors_exact(0):
        pytest.skip("host numpy exp differs from the device prior")
    H, Y, s2 = _observations("C1", 6, 2.0, 17)
    Y[0, :3] = [np.nan, np.inf, -np.inf]
    Y[1, 5] = np.nan
    Y[2, 7:9] = [np.inf, np.inf]
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=6) as dec:
        for schedule in ("stream", "onchip", "grid"):
            with np.errstate(all="ignore"):
                host = dec.decode_priors(priors_awgn_batch(Y, s2), 10, schedule=schedule)
            _assert_same(dec.decode_batch(Y, s2, 10, schedule=schedule), host)
