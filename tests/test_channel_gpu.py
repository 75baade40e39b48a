"""f1 device channel: integer-exact RNG streams, device Box-Muller (statistical parity with the reference)."""

import numpy as np
import pytest

from conftest import GOLDEN, golden_code
from paper_1609_01567_b200 import channel as ch

pytestmark = pytest.mark.gpu


def test_device_noise_matches_reference_stream(cuda):
    import torch

    from paper_1609_01567_b200 import _native

    g = np.load(GOLDEN / "channel.npz")
    ref = g["channel/y_h96_seed5"]                     # reference transmit_all_zero, frames 0..5, point 0
    y = torch.empty((6, 96), dtype=torch.float64, device="cuda")
    _native.check(_native.lib().ldpc_channel_awgn(5, 0, 0, 6, 96, 0.63, y.data_ptr(), None))
    torch.cuda.synchronize()
    d = np.abs(y.cpu().numpy() - ref)
    assert d.max() <= 1e-13, d.max()                   # same uniforms; device log/sincos within a few ulp
    # longer (odd-length) frames across several 256-draw jump segments, other points: vs the host exact path
    for n in (1001, 6145):
        states = [ch.derive_state(123, 2, f) for f in range(7, 10)]
        host = ch.transmit_all_zero_batch(n, 0.8, states, exact=True)
        y2 = torch.empty((3, n), dtype=torch.float64, device="cuda")
        _native.check(_native.lib().ldpc_channel_awgn(123, 2, 7, 3, n, 0.8, y2.data_ptr(), None))
        torch.cuda.synchronize()
        assert np.abs(y2.cpu().numpy() - host).max() <= 1e-12, n


@pytest.mark.parametrize("name", ["h96", "h14"])
def test_device_sweep_statistically_matches_reference(cuda, golden_tables, name):
    g = np.load(GOLDEN / "channel.npz")
    H = golden_code(golden_tables, name)
    frames, it, seed = (int(x) for x in g[f"ber/{name}/args"])
    pts = ch.ber_sweep(H, g[f"ber/{name}/ebno"], frames, max_iterations=it, seed=seed, batch=16, channel="device")
    ref = g[f"ber/{name}/points"]
    for p, r in zip(pts, ref):
        assert p.frames == int(r[2]) and p.sigma2 == r[1]
        assert abs(p.bit_errors - int(r[3])) <= max(3, 0.05 * r[3])
        assert abs(p.failures - int(r[6])) <= max(1, 0.05 * r[6])


def test_device_sweep_large_code_close_to_host_channel(cuda):
    """C1 code, 256 frames at 1.5 dB: device channel vs the exact host channel, same seeds."""
    from paper_1609_01567_b200 import configs

    H = configs.code("C1")
    a = ch.ber_sweep(H, [1.5], 256, max_iterations=30, seed=3, batch=128, channel="device")[0]
    b = ch.ber_sweep(H, [1.5], 256, max_iterations=30, seed=3, batch=128, exact_channel=True)[0]
    assert abs(a.failures - b.failures) <= 3
    assert abs(a.mean_iterations - b.mean_iterations) <= 0.2


def test_c_abi_error_count_allreduce_single_rank(cuda):
    # G6 through the C ABI (NCCL loaded on first use): a one-rank communicator sums in place
    import ctypes

    import torch

    from paper_1609_01567_b200 import _native

    L = _native.lib()
    uid = (ctypes.c_uint8 * 128)()
    _native.check(L.ldpc_comm_unique_id(uid), "ldpc_comm_unique_id")
    comm = ctypes.c_void_p()
    _native.check(L.ldpc_comm_create(1, 0, uid, ctypes.byref(comm)), "ldpc_comm_create")
    try:
        counts = torch.tensor([3054220, 66560, 665600, 66560], dtype=torch.int64, device="cuda")
        _native.check(L.ldpc_allreduce_counts_i64(comm, ctypes.c_void_p(counts.data_ptr()), 4,
                                                  _native.current_stream_handle()), "allreduce")
        torch.cuda.synchronize()
        assert counts.tolist() == [3054220, 66560, 665600, 66560]
        with pytest.raises(ValueError):
            _native.check(L.ldpc_comm_create(2, 2, uid, ctypes.byref(ctypes.c_void_p())), "bad rank")
    finally:
        L.ldpc_comm_destroy(comm)
