"""Pins of oracle.perf_model (Eqs. 1-7) and oracle.flops."""
import json
import os
from fractions import Fraction
from math import inf

import pytest

from oracle import flops, grid, perf_model as pm

GOLD = os.path.join(os.path.dirname(__file__), "golden")
GB = 1e11


def test_eq7_paper_cases():
    g = json.load(open(os.path.join(GOLD, "paper_eq7_cases.json")))
    beta_inter = 25e9
    for c in g["cases"]:
        cfg = tuple(c["cfg"])
        betas = pm.effective_bandwidths(cfg, c["g_node"], pm.uniform_table(c["g_node"], 1e12), beta_inter)
        assert betas[c["level"]] == pytest.approx(beta_inter * c["beta_over_beta_inter"], rel=0)
        if "ring_members" in c:
            assert [list(z) for z in grid.groups(cfg, "z")] == c["ring_members"]


def test_case1_table_lookup_and_missing_key():
    table = {(1, 2): 300e9, (2, 2): 200e9, (4, 2): 100e9, (1, 4): 250e9, (2, 4): 150e9}
    b = pm.effective_bandwidths((2, 2, 2, 1), 8, table, 25e9)
    assert b == (300e9, 200e9, 100e9, inf)
    with pytest.raises(KeyError, match="G0=1, G1=8"):
        pm.effective_bandwidths((8, 1, 1, 1), 8, table, 25e9)
    # level crossing the node: Case 2 even when the table has entries
    b = pm.effective_bandwidths((2, 2, 2, 2), 8, table, 24e9)
    assert b[3] == 24e9 / 8


def test_spec_worked_value():
    # k=n=8192, (2,2,2), b=2, β_z = 100 GB/s -> t_AG,z ≈ 1.678e-4 s
    L = pm.Layer(8192, 8192, 8192)
    t = pm.layer_times(L, (2, 2, 2, 1), (GB, GB, GB, inf))
    assert float(t["ag_z"]) == pytest.approx(1.678e-4, rel=1e-3)
    assert pm.layer_bytes(L, (2, 2, 2, 1))["ag_z"] == 16777216


def test_singletons_and_identities():
    L = pm.Layer(1024, 512, 768)
    for cfg in grid.enumerate_configs(16):
        if not pm.feasible(L, cfg):
            continue
        byts = pm.layer_bytes(L, cfg)
        gx, gy, gz, gd = cfg
        if gz == 1:
            assert byts["ag_z"] == 0 and byts["rs_z"] == 0
        if gd == 1:
            assert byts["ar_d"] == 0
        if gy == 1:
            assert byts["ar_y"] == 0
        if gx == 1:
            assert byts["ar_x"] == 0
        t = pm.layer_times(L, cfg, (GB, GB, GB, GB))
        assert t["comm"] == sum(t[k] for k in ("ag_z", "rs_z", "ar_y", "ar_x", "ar_d"))
        # transposed-layer involution
        Lt = pm.Layer(L.m, L.k, L.n, True)
        assert pm.layer_bytes(Lt, (gx, gy, gz, gd)) == pm.layer_bytes(L, (gy, gx, gz, gd))


def test_z_versus_data_tie():
    # R12: with equal β, (Gx,Gy,p,1) and (Gx,Gy,1,p) cost the same
    L = pm.gpt_block(4096, 16384)
    for p in (2, 4):
        a = pm.network_times(L, (1, 1, p, 1), (GB,) * 4)["comm"]
        b = pm.network_times(L, (1, 1, 1, p), (GB,) * 4)["comm"]
        assert a == b


def test_ranking_invariant_to_bandwidth_scale():
    L = pm.gpt_block(7168, 16384)
    t1 = {(1, 2): 300e9, (2, 2): 200e9, (4, 2): 100e9, (1, 4): 250e9, (2, 4): 150e9, (1, 8): 90e9}
    t2 = {k: 4 * v for k, v in t1.items()}
    r1 = [c for c, _ in pm.rank_configs(L, 8, 8, t1, 25e9)]
    r2 = [c for c, _ in pm.rank_configs(L, 8, 8, t2, 100e9)]
    assert r1 == r2


def test_infeasible_raises():
    with pytest.raises(ValueError, match="infeasible"):
        pm.rank_configs([pm.Layer(3, 5, 7)], 2, 8, pm.uniform_table(8, GB), GB)


def test_gpt_block_reproduces_table2_parameter_counts():
    # 12h² weights per block x layers ≈ the parameter counts of Table II
    g = json.load(open(os.path.join(GOLD, "paper_table2.json")))
    for name, pb, layers, h, heads in g["rows"]:
        w = sum(L.k * L.n for L in pm.gpt_block(h, 1)) * layers
        assert abs(w / 1e9 - pb) / pb < 0.08, name


def test_survey_80b_g8_ranking():
    # Phase A, Gd = 1, uniform β: GB per GPU per block (SURVEY.md §8(c) derived list)
    expect = [((4, 1, 2, 1), 2.114), ((4, 2, 1, 1), 2.416), ((2, 2, 2, 1), 2.517),
              ((8, 1, 1, 1), 2.819), ((2, 1, 4, 1), 3.121), ((1, 2, 4, 1), 3.926),
              ((2, 4, 1, 1), 4.027), ((1, 4, 2, 1), 4.530), ((1, 1, 8, 1), 6.342),
              ((1, 8, 1, 1), 8.456)]
    L = pm.gpt_block(12288, 16384)
    ranked = pm.rank_configs(L, 8, 8, pm.uniform_table(8, 1e9), 1e9, fixed_gd=1)
    got = [(c, round(float(t["comm"]), 3)) for c, t in ranked]
    assert got == expect


def test_c3_appendix_bytes():
    # SURVEY.md appendix C3 (20B, 2x2x2): per-layer MB sent per GPU, phase A
    L = pm.gpt_block(7168, 16384)
    want = [312.0, 143.1, 396.4, 396.4]
    for layer, w in zip(L, want):
        tot = sum(pm.layer_bytes(layer, (2, 2, 2, 1)).values())
        assert round(float(tot) / 1e6, 1) == w


# ---------------------------------------------------------------- flops

def test_flops_small_and_recompute():
    assert flops.layer_flops(2, 2, 2) == 48
    assert flops.layer_flops(3, 5, 7, recompute=True) * 6 == flops.layer_flops(3, 5, 7) * 8
    assert flops.network_flops([]) == 0


def test_table3_efficiency_arithmetic():
    g = json.load(open(os.path.join(GOLD, "paper_table3.json")))
    for system, gpus, model, pf, adv, emp in g["rows"]:
        pk = g["peaks_tflops"][system]
        e = flops.efficiency(pf * 1e15, gpus, pk["advertised"] * 1e12, pk["empirical"] * 1e12)
        assert abs(e["pct_advertised"] - adv) <= 0.2, (system, gpus)
        assert abs(e["pct_empirical"] - emp) <= 0.2, (system, gpus)


def test_mixed_precision_hand_values():
    # Eqs. 2 and 5 with b = 4 on a layer small enough to do by hand:
    # k = n = 8, Gz = Gd = 2, Gx = Gy = 1, m = 8.
    #   Eq. 2: (Gz-1)/Gz * k n /(Gx Gy) * 4       = 1/2 * 64 * 4        = 128
    #   Eq. 5: 2 (Gd-1)/Gd * k n /(Gx Gy Gz) * 4  = 2 * 1/2 * 32 * 4    = 128
    #   Eq. 1 stays bf16: (Gz-1) * k n/(Gx Gy Gz) * 2 = 32 * 2          = 64
    L = pm.Layer(8, 8, 8, False)
    by = pm.layer_bytes(L, (1, 1, 2, 2), b=2, b_grad=4)
    assert by["rs_z"] == 128 and by["ar_d"] == 128 and by["ag_z"] == 64
    assert by["ar_y"] == 0 and by["ar_x"] == 0
    # b_grad = b is the paper's single-precision form
    assert pm.layer_bytes(L, (1, 1, 2, 2), b=2, b_grad=2) == pm.layer_bytes(L, (1, 1, 2, 2), b=2)


def test_fp32_gradients_shift_the_ranking_toward_tensor_parallelism():
    # doubling only the gradient bytes makes Z/DATA (whose cost is all
    # gradient for DATA, half for Z) relatively dearer: the all-DATA config
    # never improves its rank
    layers = pm.gpt_block(4096, 16384, "A")
    tb = pm.uniform_table(8, GB)
    r2 = [c for c, _ in pm.rank_configs(layers, 8, 8, tb, GB, b=2)]
    r4 = [c for c, _ in pm.rank_configs(layers, 8, 8, tb, GB, b=2, b_grad=4)]
    assert sorted(r2) == sorted(r4)
    assert r4.index((1, 1, 1, 8)) >= r2.index((1, 1, 1, 8))


def test_gpt_block_rejects_unknown_phase():
    # reading R2b names exactly two phases; anything else is a caller error,
    # not a silent phase B
    with pytest.raises(ValueError, match="phase"):
        pm.gpt_block(4096, 16384, "fwd")
    assert [L.transposed for L in pm.gpt_block(64, 8, "B")] == [True, False, True, False]


@pytest.mark.parametrize("cfg,g_node,want", [
    # Case 1 while prod_{j<=i} G_j <= g_node, else Eq. 7: beta_inter / min(g_node, prod_{j<i} G_j)
    ((2, 2, 2, 2), 4, ("T12", "T22", "B/4", "B/4")),
    ((8, 1, 1, 1), 4, ("B/1", "inf", "inf", "inf")),
    ((1, 2, 4, 2), 2, ("inf", "T12", "B/2", "B/2")),
    ((2, 1, 1, 8), 1, ("B/1", "inf", "inf", "B/1")),
    ((4, 2, 2, 1), 8, ("T14", "T42", "B/8", "inf")),
    ((2, 4, 2, 2), 8, ("T12", "T24", "B/8", "B/8")),
    ((1, 1, 4, 4), 2, ("inf", "inf", "B/1", "B/2")),
])
def test_eq7_hand_computed_case2_betas(cfg, g_node, want):
    """Eq. 7 on grids that span nodes, each beta worked by
    hand from the hierarchy products (X, Y, Z, DATA innermost first)."""
    B = 100e9
    T = {(1, 2): 510e9, (2, 2): 470e9, (1, 4): 630e9, (4, 2): 300e9, (2, 4): 280e9,
         (1, 8): 700e9}
    hand = {"inf": inf, "T12": T[(1, 2)], "T22": T[(2, 2)], "T14": T[(1, 4)], "T42": T[(4, 2)],
            "T24": T[(2, 4)], "B/1": B, "B/2": B / 2, "B/4": B / 4, "B/8": B / 8}
    assert pm.effective_bandwidths(cfg, g_node, T, B) == tuple(hand[w] for w in want)
