"""CPU checks of the C-ABI library: it loads, exports every symbol include/axonn.h
declares, and its pure-host logic (grid bijection, groups, shard geometry,
performance model) agrees with the oracle.  No compute calls (no GPU here)."""
import os
import re

import pytest

import paper_2502_08145_b200 as ax
from oracle import alg1, grid, perf_model as pm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "axonn.h")).read()
    return sorted(set(re.findall(r"\b(axonn_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(ax._lib, s), s            # exported by libaxonn.so
        assert s in ax.EXPORTED, s               # bound with a prototype in the binding
        assert hasattr(ax, s), s                 # same name in Python


def test_version_and_error_string():
    assert ax.axonn_version() >= 100
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_rank_to_coords(0, (0, 1, 1, 1))
    assert e.value.status == ax.AXONN_ERR_CONFIG
    assert "configuration error" in ax.axonn_last_error()


@pytest.mark.parametrize("cfg", [(2, 2, 2, 2), (1, 4, 2, 1), (3, 1, 2, 2), (1, 1, 1, 1)])
def test_coords_and_groups_match_oracle(cfg):
    G = cfg[0] * cfg[1] * cfg[2] * cfg[3]
    for r in range(G):
        assert ax.axonn_rank_to_coords(r, cfg) == grid.rank_to_coords(r, cfg)
        for a in "xyzd":
            assert ax.axonn_group_members(r, cfg, a) == grid.group_of(r, cfg, a)


@pytest.mark.parametrize("transposed", [False, True])
def test_shard_geometry_matches_oracle(transposed):
    m, k, n = 96, 48, 72
    for G in (1, 2, 4, 8, 12):
        for cfg in grid.enumerate_configs(G):
            if not pm.feasible(pm.Layer(m, k, n, transposed), cfg):
                with pytest.raises(ax.AxonnError) as e:
                    ax.axonn_shard_geometry(m, k, n, cfg, 0, transposed)
                assert e.value.status == ax.AXONN_ERR_SHAPE
                continue
            for r in range(G):
                g = ax.axonn_shard_geometry(m, k, n, cfg, r, transposed)
                o = alg1.geometry(m, k, n, cfg, r, transposed)
                assert tuple(g) == (o.m_l, o.k_l, o.n_l, o.row0, o.in_col0, o.out_col0,
                                    o.what_off, o.what_len)


def test_shape_error_names_axis():
    with pytest.raises(ax.AxonnError, match="Gy"):
        ax.axonn_shard_geometry(8, 5, 8, (1, 2, 1, 1), 0)


def _table(g_node):
    # a non-uniform Case-1 database: bandwidth falls with group size and depth
    return {(g0, g1): 400e9 / (g1 ** 0.5) / (1 + 0.1 * g0)
            for g0 in range(1, g_node + 1) for g1 in range(2, g_node + 1) if g0 * g1 <= g_node}


@pytest.mark.parametrize("G,g_node,h,phase,gd", [(8, 8, 12288, "A", 1), (8, 8, 7168, "B", 0),
                                                 (16, 4, 9216, "A", 0), (32, 4, 7168, "A", 1),
                                                 (4, 8, 4096, "A", 0), (2, 8, 4096, "B", 0),
                                                 (64, 8, 16384, "A", 0)])
def test_grid_select_matches_oracle(G, g_node, h, phase, gd):
    layers = pm.gpt_block(h, 16384, phase)
    tb = _table(g_node)
    want = pm.rank_configs(layers, G, g_node, tb, 25e9, b=2, fixed_gd=gd)
    got = ax.axonn_grid_select([(L.m, L.k, L.n, L.transposed) for L in layers], G, g_node, tb,
                               25e9, 2, gd)
    assert [(r["gx"], r["gy"], r["gz"], r["gd"]) for r in got] == [c for c, _ in want]
    for r, (_, t) in zip(got, want):
        for key, ok in (("t_ag_z", "ag_z"), ("t_rs_z", "rs_z"), ("t_ar_y", "ar_y"),
                        ("t_ar_x", "ar_x"), ("t_ar_data", "ar_d"), ("t_comm", "comm")):
            assert r[key] == pytest.approx(float(t[ok]), rel=1e-12, abs=0)


@pytest.mark.parametrize("G,gd", [(8, 0), (16, 2), (64, 0)])
def test_grid_select_mp_matches_oracle(G, gd):
    layers = pm.gpt_block(6144, 16384, "A")
    tb = _table(8)
    want = pm.rank_configs(layers, G, 8, tb, 25e9, b=2, fixed_gd=gd, b_grad=4)
    got = ax.axonn_grid_select([(L.m, L.k, L.n, L.transposed) for L in layers], G, 8, tb,
                               25e9, 2, gd, grad_bytes_per_elem=4)
    assert [(r["gx"], r["gy"], r["gz"], r["gd"]) for r in got] == [c for c, _ in want]
    for r, (_, t) in zip(got, want):
        for key, ok in (("t_ag_z", "ag_z"), ("t_rs_z", "rs_z"), ("t_ar_y", "ar_y"),
                        ("t_ar_x", "ar_x"), ("t_ar_data", "ar_d"), ("t_comm", "comm")):
            assert r[key] == pytest.approx(float(t[ok]), rel=1e-12, abs=0)


def test_grid_select_errors():
    L = [(3, 5, 7, False)]
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_grid_select(L, 2, 8, pm.uniform_table(8, 1e9), 1e9)
    assert e.value.status == ax.AXONN_ERR_INFEASIBLE
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_grid_select([(64, 64, 64, False)], 4, 8, {}, 1e9)
    assert e.value.status == ax.AXONN_ERR_CONFIG and "G0=1, G1=" in str(e.value)


def test_chain_plan_and_layouts_on_every_grid():
    """The chained block bench.py times: every non-external
    input is the previous layer's output shard, byte for byte, on every grid of
    up to 16 ranks — checked through the ABI's host geometry."""
    from bench import block_layers, chain_plan
    assert chain_plan(4) == ([0, 1], [3, 0])
    assert chain_plan(8) == ([0, 1, 5], [7, 4, 0])
    assert chain_plan(4, chain=False) == ([0, 1, 2, 3], [3, 2, 1, 0])
    layers = block_layers(64, 256) * 2          # two blocks, h = 64, m = 256
    ext_I, ext_dO = chain_plan(len(layers))
    checked = 0
    for G in (1, 2, 4, 8, 16):
        for cfg in grid.enumerate_configs(G):
            if not all(pm.feasible(pm.Layer(*L), cfg) for L in layers):
                continue
            for r in range(G):
                geo = [ax.axonn_shard_geometry(m, k, n, cfg, r, t) for (m, k, n, t) in layers]
                for i in range(len(layers)):
                    if i not in ext_I:      # I_i == O_{i-1}: same rows, same columns
                        p, g = geo[i - 1], geo[i]
                        assert (p.m_l, p.row0, p.n_l, p.out_col0) == (g.m_l, g.row0, g.k_l, g.in_col0)
                    if i not in ext_dO:     # dO_i == dI_{i+1}
                        q, g = geo[i + 1], geo[i]
                        assert (q.m_l, q.row0, q.k_l, q.in_col0) == (g.m_l, g.row0, g.n_l, g.out_col0)
            checked += 1
    assert checked > 30


def test_argument_and_state_errors_without_a_device():
    """Calls that must fail before touching a GPU: the documented error kinds
    (include/axonn.h) come back with a message, on a host with no device."""
    def status(fn, *a):
        with pytest.raises(ax.AxonnError) as e:
            fn(*a)
        assert str(e.value)           # every failure carries a message
        return e.value.status

    # grid arguments: a zero factor is a configuration error
    assert status(ax.axonn_rank_to_coords, 0, (0, 1, 1, 1)) == ax.AXONN_ERR_CONFIG
    assert status(ax.axonn_rank_to_coords, 5, (2, 1, 1, 2)) == ax.AXONN_ERR_ARG
    try:
        ax.axonn_grid_coords()
        have_grid = True          # a GPU module in this process created one
    except ax.AxonnError:
        have_grid = False
    if not have_grid:
        # no grid yet: a layer handle is a state error
        assert status(ax.axonn_fc_create, 64, 64, 64) == ax.AXONN_ERR_STATE
        assert status(ax.axonn_grid_coords) == ax.AXONN_ERR_STATE
        # a multi-rank grid needs bootstrap first
        assert status(ax.axonn_grid_init, 2, 1, 1, 1) == ax.AXONN_ERR_STATE
    # local-product argument checks precede any device access (stream 0: no torch CUDA)
    g = lambda *a: ax.axonn_gemm(*a, 0)  # noqa: E731
    assert status(g, 3, ax.AXONN_BF16, 8, 8, 8, 0, 8, 0, 8, 0, 8) == ax.AXONN_ERR_ARG
    assert status(g, 0, 7, 8, 8, 8, 0, 8, 0, 8, 0, 8) == ax.AXONN_ERR_ARG
    assert status(g, 0, ax.AXONN_BF16, -1, 8, 8, 0, 8, 0, 8, 0, 8) == ax.AXONN_ERR_ARG
    assert status(g, 0, ax.AXONN_BF16, 8, 8, 8, 0, 8, 0, 8, 0, 8) == ax.AXONN_ERR_ARG
    assert status(g, 0, ax.AXONN_BF16, 8, 16, 8, 1 << 20, 8, 1 << 20, 8, 1 << 20, 16) \
        == ax.AXONN_ERR_ARG           # ldb < N
    # geometry: bad dtype, negative sizes
    assert status(ax.axonn_shard_geometry, 64, 64, 64, (1, 1, 1, 1), 0, False, 9) == ax.AXONN_ERR_ARG
    assert status(ax.axonn_shard_geometry, -1, 64, 64, (1, 1, 1, 1), 0) == ax.AXONN_ERR_ARG
    assert status(ax.axonn_shard_geometry, 64, 64, 64, (2, 1, 1, 1), 2) == ax.AXONN_ERR_ARG
    # the grid-select mixed-precision entry validates its byte sizes
    assert status(ax.axonn_grid_select_mp, [(64, 64, 64, False)], 2, 8,
                  pm.uniform_table(8, 1e9), 1e9, 2, 0) == ax.AXONN_ERR_ARG


def test_header_is_plain_c_and_links(tmp_path):
    """include/axonn.h is a C ABI: a C99 program compiles against it with
    -Wall -Werror, links to libaxonn.so, and calls pure-host entry points
    (version, rank <-> coordinates, shard geometry, grid_select, the fused
    reduction mode, the stream-K decomposition) — no torch,
    no C++."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2502_08145_b200")
    src = tmp_path / "t.c"
    src.write_text(r'''
#include <stdio.h>
#include "axonn.h"
int main(void) {
  int c[4];
  axonn_fc_desc_t d = {4096, 1024, 512, 1, AXONN_BF16, 1, AXONN_ACT_NONE};
  axonn_geometry_t g;
  axonn_layer_t L = {16384, 4096, 4096, 0};
  axonn_bw_entry_t tb = {1, 2, 1e11};
  axonn_grid_score_t out[4];
  int n = 0;
  if (axonn_version() <= 0) return 1;
  if (axonn_rank_to_coords(13, 2, 2, 2, 2, c) != AXONN_OK) return 2;
  if (c[0] != 1 || c[1] != 0 || c[2] != 1 || c[3] != 1) return 3;
  if (axonn_shard_geometry(&d, 2, 2, 1, 1, 3, &g) != AXONN_OK) return 4;
  if (axonn_grid_select(&L, 1, 2, 8, &tb, 1, 1e11, 2, 0, out, 4, &n) != AXONN_OK || n != 4) return 5;
  if (axonn_gemm(9, AXONN_BF16, 8, 8, 8, 0, 8, 0, 8, 0, 8, 0) != AXONN_ERR_ARG) return 6;
  {
    char mode[32];
    int tile[4], role[4], k0[4], k1[4], m = 0;
    if (axonn_fused_mode(2, 2, 8192, 10752, 3584, mode, 32) != AXONN_OK) return 7;
    if (axonn_stream_k_items(128, 256, 0, 74, tile, role, k0, k1, 4, &m) != AXONN_OK || m < 1)
      return 8;
    printf("%s ", mode);
  }
  printf("ok %d %lld %lld %d%d%d%d\n", axonn_version(), (long long)g.k_l, (long long)g.n_l,
         out[0].gx, out[0].gy, out[0].gz, out[0].gd);
  return 0;
}
''')
    exe = tmp_path / "t"
    cc = subprocess.run([gcc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-I",
                         os.path.join(root, "include"), str(src), "-L", libdir, "-laxonn",
                         f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert run.returncode == 0 and "ok" in run.stdout, (run.returncode, run.stdout, run.stderr)
    words = run.stdout.split()
    assert words[0] == "red_add_pair"  # the 2-rank short-K default (axonn_fused_mode)
    # transposed layer on (2,2,1,1): k_l = k/Gx, n_l = n/Gy (R2)
    assert words[words.index("ok") + 2:words.index("ok") + 4] == ["512", "256"]
