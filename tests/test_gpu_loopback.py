"""The fused collectives of the multi-GPU path, checked on ONE GPU
(axonn_loopback_step, include/axonn.h "Test support").

axonn_loopback_step runs Alg. 1 for every rank of a grid on this device with
the multi-GPU path's own device code for every cross-rank transfer: the GEMM
epilogue's multimem.red (kMcRed) and scatter-to-owner (kScatter) modes, the
owner phase k_owner_reduce (bf16 and fp32; broadcast by multimem.st or by
plain stores to the peer; re-scatter to the DATA owners for the data-parallel
sum behind RS_z), and the Z all-gather by copy engines or by the SM pull
kernel.  Each rank's results are compared with oracle.alg1.simulate's result
for that rank (SURVEY.md §8(a) a2 AG_z, a4 AR_y, a7 AR_x, a9 RS_z, a10
AR_data, a11 the transposed layer's X<->Y swap; Alg. 1 lines 2, 4, 12, 14,
PAPER.md:375-390; data parallelism PAPER.md:313-317):

* integer inputs: bit-exact against the reduction with the path's rounding
  points (reading R8): each rank's partial product rounded to the output
  dtype, summed exactly, rounded once — and the unrounded sum of those
  partials is asserted to BE the oracle's per-rank result, so the expectation
  is the oracle's, with the rounding placed where the paper's bf16 training
  places it.  AXONN_BF16_GRADF32: dŴ is fp32 end to end, so it equals the
  oracle's dŴ exactly;
* uniform inputs: normwise error <= 2e-2 (north_star) against the oracle's
  fp64 per-rank O, dI, dŴ;
* every member of a reduction group holds bit-identical bits.
Grids: every factorisation of G = 2, 3, 4, 6, 8 (P = 2, 3, 4, 6, 8 rank
axes), normal and transposed, all three 2-rank modes (exchange of whole
partials, multimem.red forced, scatter + owner phase), both AG_z paths.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import synthdata
from oracle import alg1, fc, grid
from gpu_util import normwise_err, require_cuda

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (m, k, n) per world size: every grid of G divides it, every shard row is a
# whole number of 16-byte units, and m_l spans ragged 128-row tiles.
SHAPES = {2: (320, 192, 320), 3: (240, 192, 240), 4: (320, 192, 320), 6: (480, 384, 480),
          8: (320, 192, 320)}


@pytest.fixture(scope="module")
def ax():
    require_cuda()
    import paper_2502_08145_b200 as ax
    yield ax


def _bf16(x):
    return synthdata.bf16_round(x).astype(np.float64)


def _dev(ax, a, dtype):
    torch = require_cuda()
    a = np.ascontiguousarray(a, dtype=np.float32)
    if dtype == torch.bfloat16:
        bits = synthdata.bf16_bits(a).view(np.int16)
        return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16).cuda()
    return torch.from_numpy(a).cuda()


def _host(t):
    return t.float().cpu().numpy().astype(np.float64)


def run_loopback(ax, m, k, n, cfg, transposed, kind, flags=0, grad_f32=False, layer_id=3):
    """Shard the seeded global tensors with the library's geometry, run every
    rank through axonn_loopback_step, return (inputs, per-rank outputs, paths)."""
    torch = require_cuda()
    X, W, dY = synthdata.layer_tensors(m, k, n, layer_id, kind=kind)
    G = int(np.prod(cfg))
    dt = ax.AXONN_BF16_GRADF32 if grad_f32 else ax.AXONN_BF16
    gdt = torch.float32 if grad_f32 else torch.bfloat16
    I, Wh, dO, O, dI, dW, geos = [], [], [], [], [], [], []
    for r in range(G):
        g = ax.axonn_shard_geometry(m, k, n, cfg, r, transposed, dt)
        geos.append(g)
        I.append(_dev(ax, X[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l], torch.bfloat16))
        Wl = np.ascontiguousarray(W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])
        Wh.append(_dev(ax, Wl.reshape(-1)[g.what_off:g.what_off + g.what_len], torch.bfloat16))
        dO.append(_dev(ax, dY[g.row0:g.row0 + g.m_l, g.out_col0:g.out_col0 + g.n_l], torch.bfloat16))
        O.append(torch.full((g.m_l, g.n_l), float("nan"), dtype=torch.bfloat16, device="cuda"))
        dI.append(torch.full((g.m_l, g.k_l), float("nan"), dtype=torch.bfloat16, device="cuda"))
        dW.append(torch.full((g.what_len,), float("nan"), dtype=gdt, device="cuda"))
    paths = ax.axonn_loopback_step(m, k, n, cfg, I, Wh, dO, O, dI, dW, transposed, dt, flags)
    outs = {r: (_host(O[r]), _host(dI[r]), _host(dW[r])) for r in range(G)}
    return (X, W, dY), outs, paths


def rounded_reductions(X, W, dY, cfg, transposed, grad_f32):
    """The oracle's per-rank results (alg1.simulate) and the same sums with
    the fused path's rounding points: every rank's partial product rounded to
    its storage dtype, the group sum exact, one final rounding (R8).  RS_z
    and the data-parallel sum behind it round once each (bf16 gradients)."""
    res = alg1.simulate(X, W, dY, cfg, transposed)
    G = int(np.prod(cfg))
    ax_f, ax_b = ("x", "y") if transposed else ("y", "x")
    loc = {r: alg1.shard(X, W, dY, cfg, r, transposed) for r in range(G)}
    geo = {r: alg1.geometry(X.shape[0], X.shape[1], W.shape[1], cfg, r, transposed) for r in range(G)}
    pO = {r: fc.fc_forward(loc[r][0], res.W_full[r]) for r in range(G)}
    pI = {r: fc.fc_backward_input(loc[r][2], res.W_full[r]) for r in range(G)}
    pW = {r: fc.fc_backward_weight(loc[r][0], loc[r][2]).reshape(-1) for r in range(G)}
    rg = (lambda a: a) if grad_f32 else _bf16   # fp32 gradients: integer sums are exact
    exp = {}
    for r in range(G):
        sO = sum(pO[q] for q in grid.group_of(r, cfg, ax_f))
        sI = sum(pI[q] for q in grid.group_of(r, cfg, ax_b))
        assert np.array_equal(sO, res.O[r]) and np.array_equal(sI, res.dI[r])
        eO = _bf16(sum(_bf16(pO[q]) for q in grid.group_of(r, cfg, ax_f)))
        eI = _bf16(sum(_bf16(pI[q]) for q in grid.group_of(r, cfg, ax_b)))
        exp[r] = [eO, eI, None]
    # line 14 then the data-parallel sum: slices of the Z owners, then DATA owners
    zsum, zexact = {}, {}
    for r in range(G):
        g = geo[r]
        sl = slice(g.what_off, g.what_off + g.what_len)
        zexact[r] = sum(pW[q][sl] for q in grid.group_of(r, cfg, "z"))
        zsum[r] = rg(sum(rg(pW[q])[sl] for q in grid.group_of(r, cfg, "z")))
    for r in range(G):
        assert np.array_equal(sum(zexact[q] for q in grid.group_of(r, cfg, "d")), res.dW_hat[r])
        # Gz = 1: zsum is the rounded partial itself; Gz > 1: the RS_z owner's
        # rounded sum, which the DATA owner sums and rounds again
        exp[r][2] = zsum[r] if cfg[3] == 1 else rg(sum(zsum[q] for q in grid.group_of(r, cfg, "d")))
    return res, exp


def _expected_paths(cfg, transposed, flags, grad_f32=False):
    """The fused paths the multi-GPU mode selection takes for these shapes
    (short K): 2-rank axes exchange whole partials (or multimem.red when
    forced, or scatter + owner phase when exchange is off), wider axes scatter."""
    ax_f, ax_b = (0, 1) if transposed else (1, 0)
    want = set()
    red2, no_x, pair = bool(flags & 1), bool(flags & 16), bool(flags & 32)
    xs = bool(flags & 256)

    def two(name, es2=True):
        if pair and es2:
            return f"{name}_pairsum"
        if xs and es2:
            return f"{name}_xsum"
        if es2 and not red2 and not (flags & 1024):
            return f"{name}_redpair"  # the default below the multimem.red threshold
        return f"{name}_red" if (red2 and es2) else (f"{name}_scatter" if no_x else f"{name}_exchange")
    for name, P in (("fwd", cfg[ax_f]), ("bwd", cfg[ax_b])):
        if P == 2:
            want.add(two(name))
        elif P > 1:
            want.add(f"{name}_scatter")
    if cfg[2] > 1:
        want.add("rs_z")
        want.add("gather_pull" if flags & 4 else "gather_copy")
        if cfg[3] > 1:
            want.add("dp_after_rs")
    elif cfg[3] == 2:
        want.add(two("dp", not grad_f32))
    elif cfg[3] > 2:
        want.add("dp_scatter")
    if "bwd_exchange" in want and (flags & 512):
        want.add("bwd_sidesum")  # dÎ's exchange summed by the dW GEMM's helper warps
    return want


def check(ax, G, cfg, transposed, kind, flags=0, grad_f32=False, shape=None):
    m, k, n = shape or SHAPES[G]
    (X, W, dY), outs, paths = run_loopback(ax, m, k, n, cfg, transposed, kind, flags, grad_f32)
    tag = f"cfg={cfg} T={transposed} {kind} flags={flags} gradf32={grad_f32}"
    want = _expected_paths(cfg, transposed, flags, grad_f32)
    assert want <= paths, f"{tag}: fused paths {sorted(paths)} lack {sorted(want - paths)}"
    res, exp = rounded_reductions(X, W, dY, cfg, transposed, grad_f32)
    ax_f, ax_b = ("x", "y") if transposed else ("y", "x")
    for r in range(G):
        O, dI, dW = outs[r]
        for name, got in (("O", O), ("dI", dI), ("dW", dW)):
            assert not np.isnan(got).any(), f"{tag}: rank {r} {name} not fully written"
        if kind == "int":
            for name, got, want_r in zip(("O", "dI", "dW"), (O, dI, dW), exp[r]):
                assert np.array_equal(got, want_r.reshape(got.shape)), \
                    f"{tag}: rank {r} {name} differs from the oracle (max |d| " \
                    f"{np.max(np.abs(got - want_r.reshape(got.shape)))})"
            if grad_f32:
                assert np.array_equal(dW, res.dW_hat[r]), f"{tag}: rank {r} fp32 dW not exact"
        else:
            for name, got, ref in (("O", O, res.O[r]), ("dI", dI, res.dI[r]),
                                   ("dW", dW, res.dW_hat[r])):
                e = normwise_err(got, ref.reshape(got.shape))
                assert e <= 2e-2, f"{tag}: rank {r} {name} normwise {e:.3e}"
        # replicas of a reduction group hold identical bits
        for name, idx, axis in (("O", 0, ax_f), ("dI", 1, ax_b)):
            for q in grid.group_of(r, cfg, axis):
                assert np.array_equal(outs[q][idx], outs[r][idx]), f"{tag}: {name} replicas {r},{q}"
        for q in grid.group_of(r, cfg, "d"):
            assert np.array_equal(outs[q][2], outs[r][2]), f"{tag}: dW replicas {r},{q}"
    return paths


CASES = [(G, cfg) for G in (2, 3, 4, 6, 8) for cfg in grid.enumerate_configs(G)]


@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("G,cfg", CASES, ids=[f"{c[0]}{c[1]}{c[2]}{c[3]}" for _, c in CASES])
def test_every_grid_integer_bit_exact(ax, G, cfg, transposed):
    # default 2-rank mode for these short K (unicast red.add into both ranks'
    # outputs, kRedPair) and the copy-engine AG_z; the exchange of whole
    # partials + local sum, and with the dW GEMM doing that sum (SideSum);
    # multimem.red forced on 2-rank axes with the SM-pull AG_z; the 2-rank
    # scatter + owner phase; the exchange summed inside the GEMM (kXSum,
    # opt-in: here the first rank of each pair leaves its sums to the sweep,
    # the second sums in the GEMM)
    nr = ax.AXONN_LB_NO_REDPAIR
    check(ax, G, cfg, transposed, "int", 0)
    check(ax, G, cfg, transposed, "int", nr)
    check(ax, G, cfg, transposed, "int", nr | ax.AXONN_LB_SIDESUM)
    check(ax, G, cfg, transposed, "int", ax.AXONN_LB_RED_ALWAYS | ax.AXONN_LB_GATHER_PULL)
    check(ax, G, cfg, transposed, "int", nr | ax.AXONN_LB_NO_EXCHANGE)
    check(ax, G, cfg, transposed, "int", ax.AXONN_LB_XSUM)
    check(ax, G, cfg, transposed, "int", ax.AXONN_LB_XSUM | ax.AXONN_LB_REVERSE)
    # the sum finished inside the epilogue (kPairSum), each rank of a pair in
    # both roles (the second arriver sums and writes both outputs)
    check(ax, G, cfg, transposed, "int", ax.AXONN_LB_PAIRSUM)
    check(ax, G, cfg, transposed, "int", ax.AXONN_LB_PAIRSUM | ax.AXONN_LB_REVERSE)
    # the pull variant: partials stay local, the second arriver reads the peer's
    check(ax, G, cfg, transposed, "int", ax.AXONN_LB_PAIRSUM | ax.AXONN_LB_PAIRPULL)
    check(ax, G, cfg, transposed, "int",
          ax.AXONN_LB_PAIRSUM | ax.AXONN_LB_PAIRPULL | ax.AXONN_LB_REVERSE)


@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("G,cfg", [(G, c) for G, c in CASES if G in (4, 6, 8)],
                         ids=[f"{c[0]}{c[1]}{c[2]}{c[3]}" for G, c in CASES if G in (4, 6, 8)])
def test_every_grid_uniform_within_tolerance(ax, G, cfg, transposed):
    check(ax, G, cfg, transposed, "uniform", ax.AXONN_LB_RED_ALWAYS)
    check(ax, G, cfg, transposed, "uniform", ax.AXONN_LB_XSUM)
    check(ax, G, cfg, transposed, "uniform", 0)


@pytest.mark.parametrize("cfg", [(1, 1, 2, 1), (1, 1, 1, 2), (1, 1, 4, 2), (1, 1, 2, 4),
                                 (2, 1, 2, 2), (1, 1, 3, 2), (1, 2, 1, 3), (1, 1, 8, 1)])
@pytest.mark.parametrize("transposed", [False, True])
def test_fp32_gradients_bit_exact(ax, cfg, transposed):
    """AXONN_BF16_GRADF32 (R17): fp32 dW epilogue, fp32 RS_z / DP owner phases."""
    G = int(np.prod(cfg))
    check(ax, G, cfg, transposed, "int", 0, grad_f32=True)
    check(ax, G, cfg, transposed, "int", ax.AXONN_LB_NO_EXCHANGE | ax.AXONN_LB_NO_REDPAIR,
          grad_f32=True)
    check(ax, G, cfg, transposed, "uniform", 0, grad_f32=True)


@pytest.mark.parametrize("cfg", [(2, 1, 1, 1), (1, 2, 1, 1), (4, 1, 1, 1), (1, 1, 1, 2),
                                 (2, 2, 2, 1), (1, 1, 2, 4)])
def test_emulated_multicast_agrees(ax, cfg):
    """Without a multicast object (red.global.add / plain stores) the results
    are the same bits (the stand-in is only used on devices without NVLS)."""
    G = int(np.prod(cfg))
    check(ax, G, cfg, False, "int", ax.AXONN_LB_RED_ALWAYS | ax.AXONN_LB_EMULATE_MC)


def test_multicast_object_used_when_available(ax):
    torch = require_cuda()
    _, _, paths = run_loopback(ax, *SHAPES[2], (1, 2, 1, 1), False, "int", ax.AXONN_LB_RED_ALWAYS)
    print("loopback multicast object:", "multicast" in paths)
    assert "fwd_red" in paths   # normal layer: the forward all-reduce runs over Y


def test_errors(ax):
    torch = require_cuda()
    # fp32 test mode reduces through NCCL: no loopback
    with pytest.raises(ax.AxonnError) as e:
        z = torch.zeros(64, device="cuda")
        ax.axonn_loopback_step(8, 8, 8, (1, 1, 1, 1), [z], [z], [z], [z], [z], [z], False,
                               ax.AXONN_F32)
    assert e.value.status == ax.AXONN_ERR_UNSUPPORTED
    # a shape whose reduction the multi-GPU path would leave to NCCL
    with pytest.raises(ax.AxonnError) as e:
        run_loopback(ax, 8, 16, 24, (3, 1, 1, 1), False, "int")   # 128 dI elements over 3 ranks
    assert e.value.status == ax.AXONN_ERR_UNSUPPORTED


@pytest.mark.parametrize("cfg", [(2, 2, 1, 1), (1, 2, 2, 1), (2, 1, 2, 2), (2, 2, 2, 1)])
def test_long_k_tile_configuration(cfg):
    """512x256 (MT=2) tiles in the fused epilogues — the configuration K >= 8192
    launches take — forced on small shapes in a subprocess (the switch is read
    once per process)."""
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import test_gpu_loopback as t, paper_2502_08145_b200 as ax\n"
        "for T in (False, True):\n"
        "    t.check(ax, %d, %r, T, 'int', 0)\n"
        "    t.check(ax, %d, %r, T, 'int', ax.AXONN_LB_RED_ALWAYS)\n"
        "    t.check(ax, %d, %r, T, 'int', ax.AXONN_LB_XSUM)\n"
        "print('MT2_OK')\n" % (ROOT, os.path.join(ROOT, "tests"), int(np.prod(cfg)), cfg,
                               int(np.prod(cfg)), cfg, int(np.prod(cfg)), cfg))
    env = dict(os.environ, AXONN_PAIR_MT_FUSED="2")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=600, cwd=ROOT)
    assert p.returncode == 0 and "MT2_OK" in p.stdout, (p.stdout + p.stderr)[-3000:]


FULL = [  # (name, h, m, grid, layers): tensor-parallel proxies of BASELINE C3/C4/C5
    ("20B-C3proxy", 7168, 8192, (2, 2, 1, 1), (0, 1, 2, 3)),
    ("40B-C5proxy", 9216, 8192, (2, 1, 1, 2), (0, 3)),
    ("80B-C4proxy", 12288, 4096, (1, 2, 2, 1), (1,)),
]


@pytest.mark.parametrize("flags", [0, 256, 1024], ids=["default", "xsum", "exchange"])
@pytest.mark.parametrize("name,h,m,cfg,which", FULL, ids=[f[0] for f in FULL])
def test_full_size_tensor_parallel(ax, name, h, m, cfg, which, flags):
    """Full-size GPT-block layers on tensor-parallel grids, every rank on this
    GPU through the fused collectives in the launch configuration the
    multi-GPU bench uses (K >= 8192 launches take 512x256 tiles and, on 2-rank
    axes, multimem.red): 1024 sampled entries per rank and output against
    exact fp64 dot products of the seeded global inputs, normwise <= 2e-2."""
    torch = require_cuda()
    layers = [(m, h, 3 * h, False), (m, h, h, True), (m, h, 4 * h, False), (m, 4 * h, h, True)]
    G = int(np.prod(cfg))
    rng = np.random.default_rng(7)
    for li in which:
        mm, k, n, T = layers[li]
        X, W, dY = synthdata.layer_tensors(mm, k, n, 200 + li)
        I, Wh, dO, O, dI, dW, geos = [], [], [], [], [], [], []
        for r in range(G):
            g = ax.axonn_shard_geometry(mm, k, n, cfg, r, T)
            geos.append(g)
            I.append(_dev(ax, X[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l], torch.bfloat16))
            Wl = np.ascontiguousarray(W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])
            Wh.append(_dev(ax, Wl.reshape(-1)[g.what_off:g.what_off + g.what_len], torch.bfloat16))
            del Wl
            dO.append(_dev(ax, dY[g.row0:g.row0 + g.m_l, g.out_col0:g.out_col0 + g.n_l],
                           torch.bfloat16))
            O.append(torch.empty((g.m_l, g.n_l), dtype=torch.bfloat16, device="cuda"))
            dI.append(torch.empty((g.m_l, g.k_l), dtype=torch.bfloat16, device="cuda"))
            dW.append(torch.empty((g.what_len,), dtype=torch.bfloat16, device="cuda"))
        paths = ax.axonn_loopback_step(mm, k, n, cfg, I, Wh, dO, O, dI, dW, T, flags=flags)
        ar = np.arange(1024)

        def sampled(A, B, rows, cols):
            # exact fp64 dot products of the sampled rows/columns only
            return fc.dot_entries(A[rows, :], B[:, cols], ar, ar)

        for r, g in enumerate(geos):
            rr = rng.integers(0, g.m_l, 1024)
            cc = rng.integers(0, g.n_l, 1024)
            got = O[r][torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda()]
            ref = sampled(X, W, g.row0 + rr, g.out_col0 + cc)
            e_o = normwise_err(_host(got), ref)
            c2 = rng.integers(0, g.k_l, 1024)
            got = dI[r][torch.from_numpy(rr).cuda(), torch.from_numpy(c2).cuda()]
            ref = sampled(dY, W.T, g.row0 + rr, g.in_col0 + c2)
            e_i = normwise_err(_host(got), ref)
            f = rng.integers(0, g.what_len, 1024)
            got = dW[r][torch.from_numpy(f).cuda()]
            wr, wc = (f + g.what_off) // g.n_l, (f + g.what_off) % g.n_l
            ref = sampled(X.T, dY, g.in_col0 + wr, g.out_col0 + wc)
            e_w = normwise_err(_host(got), ref)
            print(f"{name} layer {li} ({mm}x{k}x{n} T={T}) rank {r}: O {e_o:.2e} dI {e_i:.2e} "
                  f"dW {e_w:.2e} paths {sorted(paths)}")
            assert max(e_o, e_i, e_w) <= 2e-2, (name, li, r, e_o, e_i, e_w)
        del I, Wh, dO, O, dI, dW, X, W, dY
        torch.cuda.empty_cache()


def check_act(ax, G, cfg, transposed, flags=0):
    """fc1's GeLU on the layer output (reading R18): O = GELU(Z), Z = the
    all-reduce of line 4; the backward runs lines 11-14 on dZ = dO ⊙ GELU'(Z).
    The oracle: alg1.simulate gives each rank's Z; the backward is simulated
    with the global dZ = dY ⊙ GELU'(X W) (oracle.act)."""
    from oracle import act
    m, k, n = SHAPES.get(G, SHAPES[2])
    (X, W, dY), outs, paths = run_loopback_act(ax, m, k, n, cfg, transposed, flags)
    Zg = fc.fc_forward(X, W)
    dZ = dY * act.gelu_grad(Zg)
    resZ = alg1.simulate(X, W, dY, cfg, transposed)
    resB = alg1.simulate(X, W, dZ, cfg, transposed)
    tag = f"act cfg={cfg} T={transposed} flags={flags}"
    for r in range(G):
        O, dI, dW = outs[r]
        for name, got, ref in (("O", O, act.gelu(resZ.O[r])), ("dI", dI, resB.dI[r]),
                               ("dW", dW, resB.dW_hat[r])):
            e = normwise_err(got, ref.reshape(got.shape))
            assert e <= 2e-2, f"{tag}: rank {r} {name} normwise {e:.3e}"
    return paths


def run_loopback_act(ax, m, k, n, cfg, transposed, flags):
    torch = require_cuda()
    X, W, dY = synthdata.layer_tensors(m, k, n, 9, kind="uniform")
    G = int(np.prod(cfg))
    I, Wh, dO, O, dI, dW = [], [], [], [], [], []
    for r in range(G):
        g = ax.axonn_shard_geometry(m, k, n, cfg, r, transposed)
        I.append(_dev(ax, X[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l], torch.bfloat16))
        Wl = np.ascontiguousarray(W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l])
        Wh.append(_dev(ax, Wl.reshape(-1)[g.what_off:g.what_off + g.what_len], torch.bfloat16))
        dO.append(_dev(ax, dY[g.row0:g.row0 + g.m_l, g.out_col0:g.out_col0 + g.n_l], torch.bfloat16))
        O.append(torch.full((g.m_l, g.n_l), float("nan"), dtype=torch.bfloat16, device="cuda"))
        dI.append(torch.full((g.m_l, g.k_l), float("nan"), dtype=torch.bfloat16, device="cuda"))
        dW.append(torch.full((g.what_len,), float("nan"), dtype=torch.bfloat16, device="cuda"))
    paths = ax.axonn_loopback_step(m, k, n, cfg, I, Wh, dO, O, dI, dW, transposed, ax.AXONN_BF16,
                                   flags, act=ax.AXONN_ACT_GELU)
    outs = {r: (_host(O[r]), _host(dI[r]), _host(dW[r])) for r in range(G)}
    return (X, W, dY), outs, paths


@pytest.mark.parametrize("cfg", [(1, 1, 1, 1), (1, 2, 1, 1), (2, 1, 1, 1), (1, 4, 1, 1),
                                 (2, 2, 1, 1), (1, 2, 2, 1), (2, 1, 2, 2), (1, 1, 2, 2)])
@pytest.mark.parametrize("transposed", [False, True])
def test_gelu_layer(ax, cfg, transposed):
    """GeLU fused into the exchange's local sum (2-rank forward axes), or the
    elementwise pass after the other forward modes; dGeLU before line 11."""
    G = int(np.prod(cfg))
    paths = check_act(ax, G, cfg, transposed, 0)
    paths_e = check_act(ax, G, cfg, transposed, ax.AXONN_LB_NO_REDPAIR)
    paths_x = check_act(ax, G, cfg, transposed, ax.AXONN_LB_XSUM)
    check_act(ax, G, cfg, transposed, ax.AXONN_LB_RED_ALWAYS)
    check_act(ax, G, cfg, transposed, ax.AXONN_LB_NO_EXCHANGE | ax.AXONN_LB_NO_REDPAIR)
    ax_f = 0 if transposed else 1
    if cfg[ax_f] == 2:
        assert "fwd_redpair" in paths and "fwd_exchange" in paths_e and "fwd_xsum" in paths_x
