"""Host-side pieces of bench.py that need no GPU: the Chrome-trace writer
(--trace) and the block / chain plans it labels."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class FakeEvent:
    """Stands in for torch.cuda.Event: a timestamp in ms."""

    def __init__(self, t_ms):
        self.t = t_ms

    def elapsed_time(self, other):
        return other.t - self.t


def test_trace_is_valid_chrome_trace(tmp_path):
    base = FakeEvent(0.0)
    nrep = 2
    # two layer phases and the sync, each rep: [start, end] pairs
    ev = {"qkv_fwd": [FakeEvent(1.0), FakeEvent(1.5), FakeEvent(10.0), FakeEvent(10.5)],
          "qkv_fwd_gemm": [FakeEvent(2.0), FakeEvent(2.4), FakeEvent(11.0), FakeEvent(11.4)],
          "sync": [FakeEvent(3.0), FakeEvent(3.01), FakeEvent(12.0), FakeEvent(12.01)]}
    path = tmp_path / "trace.json"
    bench.write_trace(str(path), None, ev, base, nrep, {"label": "C3 proxy", "grid": (2, 2, 1, 1)})
    d = json.load(open(path))
    evs = [e for e in d["traceEvents"] if e["ph"] == "X"]
    assert len(evs) == 3 * nrep
    assert any(e["ph"] == "M" and e["args"]["name"] == "rank 0" for e in d["traceEvents"])
    by = {(e["name"], e["args"]["rep"]): e for e in evs}
    # microseconds relative to the base event, durations from the pairs
    assert by[("qkv_fwd", 0)]["ts"] == 1000.0 and by[("qkv_fwd", 0)]["dur"] == 500.0
    assert by[("qkv_fwd", 1)]["ts"] == 10000.0
    assert by[("qkv_fwd_gemm", 1)]["cat"] == "gemm_only"
    assert by[("sync", 0)]["cat"] == "sync" and by[("qkv_fwd", 0)]["cat"] == "alg1"
    assert d["otherData"]["grid"] == [2, 2, 1, 1]


def test_block_layers_phases():
    a = bench.block_layers(4096, 16384, "A")
    b = bench.block_layers(4096, 16384, "B")
    assert [t for *_, t in a] == [False, True, False, True]
    assert [t for *_, t in b] == [True, False, True, False]
    # Table II shapes: QKV h->3h, proj h->h, fc1 h->4h, fc2 4h->h
    assert [(k, n) for _, k, n, _ in a] == [(4096, 12288), (4096, 4096), (4096, 16384), (16384, 4096)]
    assert bench.model_flops(a) == sum(6 * 16384 * k * n for _, k, n, _ in a)


def test_measured_table_grid_choice_matches_the_oracle():
    """bench's grid choice for the data-parallel line and --model runs
    (model_top1: axonn_grid_select over the measured Case-1 table in
    profiles/, missing entries at their mean) agrees with oracle.perf_model's
    ranking over the same table, for the 5B / 20B / 80B blocks at 2, 4, 8 GPUs."""
    import paper_2502_08145_b200 as ax
    from oracle import perf_model as pm
    table, src = bench.case1_table()
    assert all(v > 0 for v in table.values())
    for model in ("5B", "20B", "80B"):
        for world in (2, 4, 8):
            layers = bench.block_layers(bench.HIDDEN[model], 16384 * world)
            got, _ = bench.model_top1(ax, layers, world)
            ref = pm.rank_configs([pm.Layer(*L) for L in layers], world, 8, table, 1.0e11)
            assert got == tuple(ref[0][0]), (model, world, got, ref[0][0], src)
            # the C++ ranking's times equal the oracle's on the top entries
            full = ax.axonn_grid_select(layers, world, 8, table, 1.0e11, 2, 0, cap=5)
            for c, (cfg, t) in zip(full, ref):
                assert (c["gx"], c["gy"], c["gz"], c["gd"]) == tuple(cfg)
                assert abs(c["t_comm"] - t["comm"]) <= 1e-12 * max(1.0, t["comm"])


def test_selection_command_reproduces_the_survey_ranking():
    """tools/axonn_select.py (the paper's offline configuration selection as a
    command) on the 80B block, G = 8, Gd = 1, uniform β, phase A: the ranking
    SURVEY.md §8(c) derives from Eqs. 1-5 (GB per GPU per block: 4x1x2 2.114 <
    4x2x1 2.416 < 2x2x2 2.517 < 8x1x1 2.819 < 2x1x4 3.121 < 1x2x4 3.926 <
    2x4x1 4.027 < 1x4x2 4.530 < 1x1x8 6.342 < 1x8x1 8.456)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import axonn_select
    rows, src = axonn_select.rank("80B", 8, fixed_gd=1, uniform=100.0)
    got = [(r["gx"], r["gy"], r["gz"]) for r in rows]
    assert got == [(4, 1, 2), (4, 2, 1), (2, 2, 2), (8, 1, 1), (2, 1, 4), (1, 2, 4), (2, 4, 1),
                   (1, 4, 2), (1, 1, 8), (1, 8, 1)]
    # uniform 100 GB/s: t_comm x β = the bytes per GPU of the block
    want_gb = [2.114, 2.416, 2.517, 2.819, 3.121, 3.926, 4.027, 4.530, 6.342, 8.456]
    for r, gb in zip(rows, want_gb):
        assert abs(r["t_comm"] * 100e9 / 1e9 - gb) < 0.0015
