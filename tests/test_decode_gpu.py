"""End-to-end decode parity (serial.py:150-178, engine.py:363-440), bit-exact.

Estimates, success flags, iteration counts and syndromes must equal the
reference's on the same priors: golden fixtures from running the reference,
the CPU oracle on batches of every BASELINE config, and size-independent
properties at full size."""

import numpy as np
import pytest

from conftest import PAIRS_14_7, golden_code
from paper_1609_01567_b200 import (
    CodeTables,
    ParallelDecoder,
    ParityCheckMatrix,
    decode_awgn,
    parallel_decode_awgn,
    priors_awgn_batch,
    syndrome,
)
from paper_1609_01567_b200 import configs

pytestmark = pytest.mark.gpu


def _frames(code, B, ebno_db, seed):
    H = configs.code(code)
    s2 = configs.ebno_to_sigma2(ebno_db, configs.rate(H))
    rng = np.random.default_rng(seed)
    return H, priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)


def test_golden_decode(cuda, golden_tables, golden_decode):
    for key in golden_decode["cases"]:
        code = str(golden_decode[f"{key}/code"])
        T = CodeTables.from_matrix(golden_code(golden_tables, code))
        it = int(golden_decode[f"{key}/max_iterations"])
        P = golden_decode[f"{key}/p"]
        with ParallelDecoder(T, max_batch=len(P)) as dec:
            res = dec.decode_priors(P, it)
        assert np.array_equal(res.estimates(), golden_decode[f"{key}/estimate"]), key
        assert np.array_equal(res.success.astype(bool), golden_decode[f"{key}/success"]), key
        assert np.array_equal(res.iterations, golden_decode[f"{key}/iterations"]), key
        assert np.array_equal(res.syndromes(), golden_decode[f"{key}/syndrome"]), key


def test_golden_fixed_iterations(cuda, golden_tables, golden_decode):
    T = CodeTables.from_matrix(golden_code(golden_tables, "c1"))
    P = golden_decode["fixed/p"]
    with ParallelDecoder(T, max_batch=len(P)) as dec:
        res = dec.decode_priors(P, int(golden_decode["fixed/max_iterations"]), early_stop=False)
    assert np.array_equal(res.estimates(), golden_decode["fixed/estimate"])
    assert np.array_equal(res.success.astype(bool), golden_decode["fixed/success"])
    assert np.array_equal(res.syndromes(), golden_decode["fixed/syndrome"])
    assert (res.iterations == 10).all()


def test_single_frame_api_matches_golden(cuda, golden_tables, golden_decode):
    # the reference's call shapes: decode_awgn / parallel_decode_awgn / ParallelDecoder.decode from y
    H = golden_code(golden_tables, "h14")
    T = CodeTables.from_matrix(H)
    for key in ("h14_s05", "h14_s10"):
        Y = golden_decode[f"{key}/y"]
        s2 = float(golden_decode[f"{key}/sigma2"])
        it = int(golden_decode[f"{key}/max_iterations"])
        with ParallelDecoder(T) as dec:
            for i, y in enumerate(Y):
                for res in (decode_awgn(y, s2, it, T, H), parallel_decode_awgn(y, s2, it, T, H),
                            dec.decode(y, s2, it)):
                    assert np.array_equal(res.estimate, golden_decode[f"{key}/estimate"][i])
                    assert res.success == bool(golden_decode[f"{key}/success"][i])
                    assert res.iterations_used == int(golden_decode[f"{key}/iterations"][i])
                    assert np.array_equal(res.syndrome, golden_decode[f"{key}/syndrome"][i])


@pytest.mark.parametrize("code,B,ebno,iters,early", [
    ("C1", 70, 2.0, 50, True),
    ("C1", 33, 1.0, 50, True),
    ("C2", 64, 2.0, 20, True),
    ("C2", 40, 1.5, 20, False),
    ("C4", 24, 3.0, 20, True),
    ("C4", 20, 1.0, 8, False),
    ("C2", 300, 1.5, 20, True),   # B >= 128, early stop: positions in difficulty order
    ("C1", 1000, 1.0, 30, True),
])
def test_batches_vs_oracle(cuda, code, B, ebno, iters, early):
    from oracle import OracleTables

    H, P = _frames(code, B, ebno, seed=B * 7 + iters)
    T = CodeTables.from_matrix(H)
    with ParallelDecoder(T, max_batch=B, sub_batch=32) as dec:
        res = dec.decode_priors(P, iters, early_stop=early)
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P, iters, fixed_iterations=not early)
    assert np.array_equal(res.estimates(), est)
    assert np.array_equal(res.success.astype(bool), ok)
    assert np.array_equal(res.iterations, its)
    assert np.array_equal(res.syndromes(), z)


def test_pinned_and_pageable_buffers_agree(cuda):
    # pageable numpy in/out goes through the decoder's pinned staging slots (several 16 MB pieces at
    # C3 size); pinned buffers are copied directly: identical results
    import torch

    from paper_1609_01567_b200.decoder import BatchResult

    H, P = _frames("C3", 160, 2.0, seed=8)
    T = CodeTables.from_matrix(H)
    n, m = H.n, H.m
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
    P_pin = pin(P.shape, torch.float64)
    P_pin[:] = P
    with ParallelDecoder(T, max_batch=160, sub_batch=64) as dec:
        pageable = dec.decode_priors(P, 6, early_stop=False)
        out = BatchResult(pin((160, (n + 31) // 32), torch.int32).view(np.uint32), pin((160,), torch.uint8),
                          pin((160,), torch.int32), pin((160, (m + 31) // 32), torch.int32).view(np.uint32), n, m)
        pinned = dec.decode_priors(P_pin, 6, early_stop=False, out=out)
        mixed = dec.decode_priors(P_pin, 6, early_stop=False)  # pinned in, pageable out
    for r in (pinned, mixed):
        assert np.array_equal(r.est_bits, pageable.est_bits) and np.array_equal(r.syn_bits, pageable.syn_bits)
        assert np.array_equal(r.success, pageable.success) and np.array_equal(r.iterations, pageable.iterations)


def test_device_path_equals_host_path(cuda):
    import torch

    H, P = _frames("C2", 96, 1.8, seed=3)
    T = CodeTables.from_matrix(H)
    with ParallelDecoder(T, max_batch=96) as dec:
        host = dec.decode_priors(P, 20)
        est, ok, its, syn = dec.decode_device(torch.from_numpy(P).cuda(), 20)
        torch.cuda.synchronize()
    assert np.array_equal(est.cpu().numpy().view(np.uint32), host.est_bits)
    assert np.array_equal(ok.cpu().numpy(), host.success)
    assert np.array_equal(its.cpu().numpy(), host.iterations)
    assert np.array_equal(syn.cpu().numpy().view(np.uint32), host.syn_bits)


def test_edge_cases(cuda):
    from oracle import OracleTables

    H = ParityCheckMatrix(14, 7, PAIRS_14_7)
    T = CodeTables.from_matrix(H)
    O = OracleTables.from_matrix(H)
    rng = np.random.default_rng(5)
    with ParallelDecoder(T, max_batch=130, sub_batch=64) as dec:
        for B in (1, 31, 32, 33, 64, 65, 130):
            P = priors_awgn_batch(-1.0 + 1.2 * rng.standard_normal((B, 14)), 0.9)
            for it in (0, 1, 7):
                for early in (True, False):
                    res = dec.decode_priors(P, it, early_stop=early)
                    est, ok, its, z = O.decode_batch(P, it, fixed_iterations=not early)
                    assert np.array_equal(res.estimates(), est), (B, it, early)
                    assert np.array_equal(res.success.astype(bool), ok), (B, it, early)
                    assert np.array_equal(res.iterations, its), (B, it, early)
                    assert np.array_equal(res.syndromes(), z), (B, it, early)
        # saturated priors (p = 0 / 1 / 0.5) survive the kernels exactly like the reference
        P = np.array([[0.0, 1.0, 0.5] * 4 + [0.0, 1.0]] * 3)
        res = dec.decode_priors(P, 5)
        est, ok, its, z = O.decode_batch(P, 5)
        assert np.array_equal(res.estimates(), est) and np.array_equal(res.iterations, its)


def test_errors_mirror_reference(cuda):
    H = ParityCheckMatrix(14, 7, PAIRS_14_7)
    T = CodeTables.from_matrix(H)
    with pytest.raises(ValueError):
        ParallelDecoder(T, group_size=0)
    with pytest.raises(ValueError):
        ParallelDecoder(T, n_threads=0)
    dec = ParallelDecoder(T)
    with pytest.raises(ValueError):
        dec.decode(np.zeros(14), 0.0, 5)
    with pytest.raises(ValueError):
        dec.decode(np.zeros(13), 1.0, 5)
    with pytest.raises(ValueError):
        dec.decode(np.zeros(14), 1.0, -1)
    dec.close()
    with pytest.raises(RuntimeError):
        dec.decode(np.zeros(14), 1.0, 5)
    with pytest.raises(ValueError):
        parallel_decode_awgn(np.zeros(14), 1.0, 5, T, ParityCheckMatrix(3, 2, ((0, 0), (0, 1), (1, 1), (1, 2))))


def test_clean_codeword_zero_iterations(cuda):
    H = ParityCheckMatrix(14, 7, PAIRS_14_7)
    T = CodeTables.from_matrix(H)
    for gain in (1.0, 0.25, 3.7):
        res = decode_awgn(np.full(14, -gain), 0.4, 50, T, H)
        assert res.success and res.iterations_used == 0 and not res.estimate.any() and not res.syndrome.any()


@pytest.mark.slow
def test_dvbs2_full_batch(cuda):
    """BASELINE config C3 at full size: 1024 codewords, fixed 10 iterations.

    Sampled codewords are compared bit-exactly with the oracle; every codeword
    is checked against size-independent properties (syndrome == H * estimate,
    success <=> zero syndrome, iteration count)."""
    from oracle import OracleTables

    H, P = _frames("C3", 1024, 2.0, seed=64800)
    T = CodeTables.from_matrix(H)
    with ParallelDecoder(T, max_batch=1024) as dec:
        res = dec.decode_priors(P, 10, early_stop=False)
    est = res.estimates()
    z = res.syndromes()
    assert np.array_equal(syndrome(est[:64], T), z[:64])
    assert np.array_equal(res.success.astype(bool), ~z.any(axis=1))
    assert (res.iterations == 10).all()
    sample = np.arange(0, 1024, 37)
    e_o, ok_o, it_o, z_o = OracleTables.from_matrix(H).decode_batch(P[sample], 10, fixed_iterations=True)
    assert np.array_equal(est[sample], e_o)
    assert np.array_equal(z[sample], z_o)
    assert np.array_equal(res.success[sample].astype(bool), ok_o)
    # early-stop mode on the same frames: the reference's semantics
    with ParallelDecoder(T, max_batch=1024) as dec:
        res2 = dec.decode_priors(P, 10, early_stop=True)
    e2, ok2, it2, z2 = OracleTables.from_matrix(H).decode_batch(P[sample], 10)
    assert np.array_equal(res2.estimates()[sample], e2)
    assert np.array_equal(res2.iterations[sample], it2)
    assert np.array_equal(res2.success[sample].astype(bool), ok2)


@pytest.mark.parametrize("name", ["h96", "h14"])
def test_ber_sweep_gpu_matches_reference(cuda, golden_tables, name):
    """channel.py:83-137 semantics on the GPU decoder: BerPoints and CSV equal the reference's."""
    from conftest import GOLDEN
    from paper_1609_01567_b200 import channel as ch

    g = np.load(GOLDEN / "channel.npz")
    H = golden_code(golden_tables, name)
    frames, it, seed = (int(x) for x in g[f"ber/{name}/args"])
    pts = ch.ber_sweep(H, g[f"ber/{name}/ebno"], frames, max_iterations=it, seed=seed, batch=8, exact_channel=True)
    arr = np.array([[p.ebno_db, p.sigma2, p.frames, p.bit_errors, p.ber, p.mean_iterations, p.failures] for p in pts])
    assert np.array_equal(arr, g[f"ber/{name}/points"])
    assert ch.ber_csv(pts) == str(g[f"ber/{name}/csv"])


def test_graph_replay_reads_fresh_inputs(cuda):
    """Repeated decodes with the same buffers replay a captured CUDA graph; results must track the inputs."""
    import torch

    from oracle import OracleTables

    H = configs.code("C1")
    T = CodeTables.from_matrix(H)
    O = OracleTables.from_matrix(H)
    B = 70
    with ParallelDecoder(T, max_batch=B) as dec:
        P_dev = torch.empty((B, H.n), dtype=torch.float64, device="cuda")
        ws = dec.workspace(B)
        outs = dec.alloc_outputs(B, P_dev.device)
        for call in range(4):  # call 0 eager, call 1 captures, calls 2-3 replay
            _, P = _frames("C1", B, 1.0 + 0.3 * call, seed=100 + call)
            P_dev.copy_(torch.from_numpy(P))
            est, ok, its, syn = dec.decode_device(P_dev, 30, early_stop=True, workspace=ws, outputs=outs)
            torch.cuda.synchronize()
            e, s, i, z = O.decode_batch(P, 30)
            from paper_1609_01567_b200 import unpack_bits

            assert np.array_equal(unpack_bits(est.cpu().numpy().view(np.uint32), H.n), e), call
            assert np.array_equal(its.cpu().numpy(), i), call
            assert np.array_equal(ok.cpu().numpy().astype(bool), s), call


def test_streaming_submit_wait_matches_sync(cuda):
    # decode_priors_async / decode_stream (two batches in flight) give decode_priors' results,
    # and those equal the oracle's, for batches of varying size and both stop modes
    import torch

    from oracle import OracleTables

    H = configs.code("C2")
    O = OracleTables.from_matrix(H)
    batches = [_frames("C2", B, 1.8, seed=40 + i)[1] for i, B in enumerate((40, 64, 17, 96, 1))]
    pinned = [torch.from_numpy(P).pin_memory().numpy() for P in batches]
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=96) as dec:
        for early in (True, False):
            sync = [dec.decode_priors(P, 20, early_stop=early) for P in batches]
            streamed = list(dec.decode_stream(pinned, 20, early_stop=early))
            pend = [dec.decode_priors_async(P, 20, early_stop=early) for P in batches[:2]]
            waited = [p.wait() for p in reversed(pend)][::-1]
            for i, (a, b) in enumerate(zip(sync, streamed)):
                assert np.array_equal(a.est_bits, b.est_bits) and np.array_equal(a.syn_bits, b.syn_bits), i
                assert np.array_equal(a.success, b.success) and np.array_equal(a.iterations, b.iterations), i
            for a, b in zip(sync, waited):
                assert np.array_equal(a.est_bits, b.est_bits) and np.array_equal(a.iterations, b.iterations)
            est, ok, its, z = O.decode_batch(batches[0], 20, fixed_iterations=not early)
            assert np.array_equal(streamed[0].estimates(), est) and np.array_equal(streamed[0].iterations, its)
            assert np.array_equal(streamed[0].syndromes(), z) and np.array_equal(streamed[0].success.astype(bool), ok)
        with pytest.raises(ValueError):
            dec.decode_priors_async(np.zeros((97, H.n)), 20)


def test_batches_larger_than_max_batch_are_pipelined(cuda):
    # B > max_batch: chunks of max_batch go two at a time through the streaming slots;
    # results equal one whole-batch call and the oracle
    from oracle import OracleTables

    H, P = _frames("C1", 150, 1.5, seed=12)
    T = CodeTables.from_matrix(H)
    with ParallelDecoder(T, max_batch=64) as small, ParallelDecoder(T, max_batch=150) as big:
        for early in (True, False):
            a = small.decode_priors(P, 30, early_stop=early)
            b = big.decode_priors(P, 30, early_stop=early)
            assert np.array_equal(a.est_bits, b.est_bits) and np.array_equal(a.syn_bits, b.syn_bits)
            assert np.array_equal(a.success, b.success) and np.array_equal(a.iterations, b.iterations)
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P, 30, fixed_iterations=True)
    assert np.array_equal(a.estimates(), est) and np.array_equal(a.iterations, its)


@pytest.mark.slow
@pytest.mark.parametrize("mode", ["fixed", "early"])
def test_c3_full_batch_timed_path_all_frames(cuda, mode):
    """The bench's timed path at its full size: C3, B = 1024, one decode_device call (whole batch,
    CUDA-graph replay on the third call), every frame bit-exact vs the oracle (serial.py:150-178,
    engine.py:363-398).  fixed: the bench workload itself (2 dB, 10 rounds, bench.py's seed);
    early: 3 dB, 30 rounds, where frames stop at different rounds."""
    import torch

    from oracle import OracleTables
    from paper_1609_01567_b200 import unpack_bits

    H = configs.code("C3")
    ebno, iters, early = (2.0, 10, False) if mode == "fixed" else (3.0, 30, True)
    s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
    rng = np.random.default_rng(1000)
    P = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((1024, H.n)), s2)
    T = CodeTables.from_matrix(H)
    with ParallelDecoder(T, max_batch=1024) as dec:
        P_dev = torch.from_numpy(P).cuda()
        ws, outs = dec.workspace(1024), dec.alloc_outputs(1024, P_dev.device)
        for _ in range(3):  # eager, capture, replay: the replayed graph is what the bench times
            dec.decode_device(P_dev, iters, early_stop=early, workspace=ws, outputs=outs)
        est, ok, its, syn = (t.cpu().numpy() for t in outs)
    e_o, ok_o, it_o, z_o = OracleTables.from_matrix(H).decode_batch(P, iters, fixed_iterations=not early)
    assert np.array_equal(unpack_bits(est.view(np.uint32), H.n), e_o)
    assert np.array_equal(ok.astype(bool), ok_o)
    assert np.array_equal(its, it_o)
    assert np.array_equal(unpack_bits(syn.view(np.uint32), H.m), z_o)
    if early:
        assert len(np.unique(it_o)) > 3, "early-stop case should spread stopping rounds"


@pytest.mark.parametrize("B", [800, 769, 895, 1000])
def test_host_decoder_any_batch_up_to_max_batch(cuda, B):
    """chunk_plan(B) for B < max_batch can merge a remainder into a sub-batch larger than
    max_batch's plan has; the per-lane workspace must cover it (C2, a streaming-schedule code)."""
    from oracle import OracleTables

    H, P = _frames("C2", B, 1.8, seed=B)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=1024) as dec:
        res = dec.decode_priors(P, 12, early_stop=True)
    sample = np.arange(0, B, 41)
    e, ok, it, z = OracleTables.from_matrix(H).decode_batch(P[sample], 12)
    assert np.array_equal(res.estimates()[sample], e)
    assert np.array_equal(res.iterations[sample], it)
    assert np.array_equal(res.success[sample].astype(bool), ok)


def test_matrix_keyed_device_tables_are_released(cuda):
    """tables cached for a ParityCheckMatrix passed where the reference takes H
    (syndrome, decode_awgn) die with the matrix (CodeTables holds no reference back to it)."""
    import gc
    import weakref

    from paper_1609_01567_b200 import decoder as D

    base = configs.code("C1")
    H = ParityCheckMatrix(base.n, base.m, np.stack([base.rows, base.cols], axis=1))
    z = syndrome(np.zeros(H.n, np.uint8), H)
    assert not z.any()
    key = id(H)
    assert dict.__contains__(D._H_TABLES, key)
    graph = weakref.ref(dict.__getitem__(D._H_TABLES, key).graph)
    del H
    gc.collect()
    assert not dict.__contains__(D._H_TABLES, key)
    assert graph() is None


@pytest.mark.parametrize("code,B,schedules", [("C1", 40, ("stream", "onchip")), ("C2", 64, ("stream", "grid")),
                                               ("C4", 6, ("stream",))])
def test_high_snr_fixed_iterations_vs_oracle(cuda, code, B, schedules):
    """5 dB, fixed 12 rounds: the messages saturate (variable-side numerators of exactly 0 over
    positive denominators) for most of the decode; every schedule gives the oracle's outputs."""
    from oracle import OracleTables

    H, P = _frames(code, B, 5.0, seed=5 + B)
    est_o, ok_o, it_o, z_o = OracleTables.from_matrix(H).decode_batch(P, 12, fixed_iterations=True)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        for schedule in schedules:
            res = dec.decode_priors(P, 12, early_stop=False, schedule=schedule)
            assert np.array_equal(res.estimates(), est_o), schedule
            assert np.array_equal(res.success.astype(bool), ok_o), schedule
            assert np.array_equal(res.iterations, it_o), schedule
            assert np.array_equal(res.syndromes(), z_o), schedule
