"""Pins of oracle.alg1 — Algorithm 1 over a grid.

Pinned against: the unsharded definition (every factorisation reproduces it,
exactly on integer inputs — SURVEY.md §8(c)), Eqs. 1-5 byte counts (exact),
the C1 per-rank byte totals worked by hand, the degenerate special cases of
PAPER.md:416-425, and the shard->gather round trip.
"""
import numpy as np
import pytest

from oracle import alg1, fc, grid, perf_model
import synthdata


def _all_cfgs(maxG):
    out = []
    for G in range(1, maxG + 1):
        out += grid.enumerate_configs(G)
    return out


@pytest.mark.parametrize("transposed", [False, True])
def test_every_factorisation_reproduces_unsharded_exactly(transposed):
    m, k, n = 48, 24, 36
    X, W, dO = synthdata.layer_tensors(m, k, n, kind="int")
    O_ref, dI_ref, dW_ref = fc.fc_layer(X, W, dO)
    tried = 0
    for cfg in _all_cfgs(16):
        L = perf_model.Layer(m, k, n, transposed)
        if not perf_model.feasible(L, cfg):
            continue
        res = alg1.simulate(X, W, dO, cfg, transposed)
        O, dI, dW = alg1.gather_outputs(res, m, k, n, cfg, transposed)
        np.testing.assert_array_equal(O, O_ref)
        np.testing.assert_array_equal(dI, dI_ref)
        np.testing.assert_array_equal(dW, dW_ref)
        tried += 1
    assert tried >= 60


def test_random_inputs_close_on_2x2x2():
    m, k, n = 256, 512, 1024            # C1 of BASELINE.json
    X, W, dO = synthdata.layer_tensors(m, k, n)
    O_ref, dI_ref, dW_ref = fc.fc_layer(X, W, dO)
    cfg = (2, 2, 2, 1)
    res = alg1.simulate(X, W, dO, cfg)
    O, dI, dW = alg1.gather_outputs(res, m, k, n, cfg)
    for a, b in ((O, O_ref), (dI, dI_ref), (dW, dW_ref)):
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


def test_gathered_weight_is_exact_copy():
    m, k, n = 16, 32, 24
    X, W, dO = synthdata.layer_tensors(m, k, n)
    cfg = (2, 2, 2, 1)
    res = alg1.simulate(X, W, dO, cfg)
    for r in range(8):
        g = alg1.geometry(m, k, n, cfg, r)
        np.testing.assert_array_equal(
            res.W_full[r], W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])


def test_c1_bytes_per_rank():
    # C1: 256x512x1024 on 2x2x2, bf16: AG 131072, RS 131072, AR_y 131072, AR_x 65536
    # (SURVEY.md §8(c) "Communication volumes", worked from Eqs. 1-4 by hand)
    m, k, n = 256, 512, 1024
    X, W, dO = synthdata.layer_tensors(m, k, n)
    res = alg1.simulate(X, W, dO, (2, 2, 2, 1))
    for r in range(8):
        assert alg1.bytes_sent(res, "ag_z", r) == 131072
        assert alg1.bytes_sent(res, "rs_z", r) == 131072
        assert alg1.bytes_sent(res, "ar_fwd", r) == 131072
        assert alg1.bytes_sent(res, "ar_bwd", r) == 65536
        assert alg1.bytes_sent(res, "ar_d", r) == 0
        total = sum(alg1.bytes_sent(res, kd, r) for kd in ("ag_z", "rs_z", "ar_fwd", "ar_bwd", "ar_d"))
        assert total == 458752


@pytest.mark.parametrize("transposed", [False, True])
def test_simulated_bytes_equal_eqs_1_to_5(transposed):
    m, k, n = 96, 48, 96
    X, W, dO = synthdata.layer_tensors(m, k, n)
    L = perf_model.Layer(m, k, n, transposed)
    for cfg in _all_cfgs(16):
        if not perf_model.feasible(L, cfg):
            continue
        # ring all-reduce pads to a multiple of p; use shapes where Eqs. 1-5 are integral
        res = alg1.simulate(X, W, dO, cfg, transposed)
        eq = perf_model.layer_bytes(L, cfg, b=2)
        gx, gy, gz, gd = cfg
        pf, pb = (gx, gy) if transposed else (gy, gx)
        g0 = alg1.geometry(m, k, n, cfg, 0, transposed)
        if (g0.m_l * g0.n_l) % pf or (g0.m_l * g0.k_l) % pb or g0.what_len % gd:
            continue
        for r in range(gx * gy * gz * gd):
            assert alg1.bytes_sent(res, "ag_z", r) == eq["ag_z"]
            assert alg1.bytes_sent(res, "rs_z", r) == eq["rs_z"]
            assert alg1.bytes_sent(res, "ar_fwd", r) == eq["ar_y"]
            assert alg1.bytes_sent(res, "ar_bwd", r) == eq["ar_x"]
            assert alg1.bytes_sent(res, "ar_d", r) == eq["ar_d"]


def test_fsdp_special_case_only_z_collectives():
    # only the Z axis -> FSDP/ZeRO: Eqs. 3-4 vanish
    m, k, n = 32, 16, 24
    X, W, dO = synthdata.layer_tensors(m, k, n)
    res = alg1.simulate(X, W, dO, (1, 1, 4, 1))
    for r in range(4):
        assert alg1.bytes_sent(res, "ar_fwd", r) == 0 and alg1.bytes_sent(res, "ar_bwd", r) == 0
        assert alg1.bytes_sent(res, "ag_z", r) > 0 and alg1.bytes_sent(res, "rs_z", r) > 0


def test_megatron_special_case():
    # X axis with the transpose scheme -> Megatron-LM 1D TP.
    # Normal layer: columns split over X, backward all-reduce only; transposed
    # layer: rows split over X, forward all-reduce only.
    m, k, n = 16, 24, 32
    X, W, dO = synthdata.layer_tensors(m, k, n)
    a = alg1.simulate(X, W, dO, (4, 1, 1, 1), transposed=False)
    b = alg1.simulate(X, W, dO, (4, 1, 1, 1), transposed=True)
    for r in range(4):
        assert alg1.bytes_sent(a, "ar_fwd", r) == 0 and alg1.bytes_sent(a, "ar_bwd", r) > 0
        assert alg1.bytes_sent(b, "ar_fwd", r) > 0 and alg1.bytes_sent(b, "ar_bwd", r) == 0
        for kd in ("ag_z", "rs_z", "ar_d"):
            assert alg1.bytes_sent(a, kd, r) == 0 and alg1.bytes_sent(b, kd, r) == 0


def test_two_layer_chain_with_transpose():
    # O of a normal layer is laid out exactly as the input of a
    # transposed layer, so the chain runs without redistribution.
    m, k, h, n = 32, 16, 24, 8
    cfg = (2, 2, 2, 1)
    X = synthdata.tensor((m, k), 101, kind="int")
    W1 = synthdata.tensor((k, h), 102, kind="int")
    W2 = synthdata.tensor((h, n), 103, kind="int")
    for r in range(8):
        g1 = alg1.geometry(m, k, h, cfg, r, transposed=False)
        g2 = alg1.geometry(m, h, n, cfg, r, transposed=True)
        assert (g1.row0, g1.out_col0, g1.n_l) == (g2.row0, g2.in_col0, g2.k_l)
    res1 = alg1.simulate(X, W1, np.zeros((m, h)), cfg, False)
    O1, _, _ = alg1.gather_outputs(res1, m, k, h, cfg, False)
    res2 = alg1.simulate(O1, W2, np.zeros((m, n)), cfg, True)
    O2, _, _ = alg1.gather_outputs(res2, m, h, n, cfg, True)
    np.testing.assert_array_equal(O2, fc.naive_matmul(fc.naive_matmul(X, W1), W2))


def test_data_parallel_sum_matches_full_batch():
    # replicas hold batch shards; all-reduce of gradients (sum, R9)
    m, k, n = 64, 16, 16
    X, W, dO = synthdata.layer_tensors(m, k, n, kind="int")
    res = alg1.simulate(X, W, dO, (1, 1, 1, 4))
    for r in range(4):
        np.testing.assert_array_equal(res.dW_hat[r], (X.T.astype(float) @ dO).reshape(-1))


def test_shape_errors_name_the_axis():
    with pytest.raises(ValueError, match="Gy"):
        alg1.check_shape(8, 5, 8, (1, 2, 1, 1))
    with pytest.raises(ValueError, match="Gx"):
        alg1.check_shape(8, 8, 5, (2, 1, 1, 1))
    with pytest.raises(ValueError, match="Gz"):
        alg1.check_shape(7, 8, 8, (1, 1, 2, 1))
    with pytest.raises(ValueError, match="Gx"):
        alg1.check_shape(8, 5, 8, (2, 1, 1, 1), transposed=True)


@pytest.mark.parametrize("transposed", [False, True])
def test_mixed_precision_bytes_equal_eqs_1_to_5(transposed):
    # reading R17: weights and activations move in bf16 (b = 2 in Eqs. 1, 3,
    # 4), the gradient reductions RS_z and AR_data in fp32 (b = 4 in Eqs. 2, 5)
    m, k, n = 64, 32, 64
    X, W, dO = synthdata.layer_tensors(m, k, n)
    L = perf_model.Layer(m, k, n, transposed)
    for cfg in [(1, 1, 2, 2), (2, 1, 2, 2), (1, 2, 4, 2), (1, 1, 1, 8), (1, 1, 8, 1)]:
        res = alg1.simulate(X, W, dO, cfg, transposed)
        eq = perf_model.layer_bytes(L, cfg, b=2, b_grad=4)
        for r in range(cfg[0] * cfg[1] * cfg[2] * cfg[3]):
            assert alg1.bytes_sent(res, "ag_z", r, 2) == eq["ag_z"]
            assert alg1.bytes_sent(res, "ar_fwd", r, 2) == eq["ar_y"]
            assert alg1.bytes_sent(res, "ar_bwd", r, 2) == eq["ar_x"]
            assert alg1.bytes_sent(res, "rs_z", r, 4) == eq["rs_z"]
            assert alg1.bytes_sent(res, "ar_d", r, 4) == eq["ar_d"]
