"""Alg. 1 through the C ABI on one GPU (grid 1x1x1x1, BASELINE.json C2's grid):
axonn_fc_forward / axonn_fc_backward / axonn_grads_sync against oracle.fc."""
import numpy as np
import pytest

import synthdata
from oracle import fc
from gpu_util import bf16_bits_of, empty_dev, normwise_err, require_cuda, to_dev, to_host_f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ax():
    require_cuda()
    import paper_2502_08145_b200 as ax
    try:
        ax.axonn_grid_init(1, 1, 1, 1)
    except ax.AxonnError as e:            # another module already created the grid
        assert e.status == ax.AXONN_ERR_STATE
    yield ax


def _layer(ax, m, k, n, transposed, kind, dtype_t, layer_id=0, grad_f32=False):
    torch = require_cuda()
    X, W, dY = synthdata.layer_tensors(m, k, n, layer_id, kind=kind)
    dt = ax.AXONN_F32 if dtype_t == torch.float32 else ax.AXONN_BF16
    if grad_f32:
        dt = ax.AXONN_BF16_GRADF32
    h = ax.axonn_fc_create(m, k, n, transposed, dt)
    g = ax.axonn_fc_geometry(h)
    assert (g.m_l, g.k_l, g.n_l, g.what_len) == (m, k, n, k * n)
    I = to_dev(X, dtype_t)
    What = to_dev(W.reshape(1, -1), dtype_t).reshape(-1)
    dO = to_dev(dY, dtype_t)
    O = empty_dev(m, n, dtype_t)
    dI = empty_dev(m, k, dtype_t)
    dW = empty_dev(1, k * n, torch.float32 if grad_f32 else dtype_t).reshape(-1)
    ax.axonn_fc_forward(h, I, What, O)
    ax.axonn_fc_backward(h, dO, dI, dW)
    ax.axonn_grads_sync()
    torch.cuda.synchronize()
    ax.axonn_fc_destroy(h)
    return (X, W, dY), (O, dI, dW.reshape(k, n))


@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("m,k,n", [(256, 512, 1024), (384, 200, 136)])
def test_integer_bit_exact(ax, m, k, n, transposed):
    torch = require_cuda()
    (X, W, dY), outs = _layer(ax, m, k, n, transposed, "int", torch.bfloat16)
    for got, ref in zip(outs, fc.fc_layer(X, W, dY)):
        want = synthdata.bf16_bits(synthdata.bf16_round(ref))
        assert np.array_equal(bf16_bits_of(got), want)


@pytest.mark.parametrize("m,k,n", [(256, 512, 1024), (2048, 1024, 3072)])
def test_random_within_tolerance(ax, m, k, n):
    torch = require_cuda()
    (X, W, dY), outs = _layer(ax, m, k, n, False, "uniform", torch.bfloat16)
    for got, ref in zip(outs, fc.fc_layer(X, W, dY)):
        assert normwise_err(to_host_f64(got), ref) <= 2e-2


def test_f32_mode_bit_exact(ax):
    torch = require_cuda()
    (X, W, dY), outs = _layer(ax, 192, 96, 160, False, "int", torch.float32)
    for got, ref in zip(outs, fc.fc_layer(X, W, dY)):
        np.testing.assert_array_equal(to_host_f64(got), ref)


@pytest.mark.parametrize("transposed", [False, True])
@pytest.mark.parametrize("m,k,n", [(256, 512, 1024), (384, 200, 136), (129, 96, 520)])
def test_grad_f32_integer_bit_exact(ax, m, k, n, transposed):
    """AXONN_BF16_GRADF32 (reading R17): O and dI as in bf16 mode, dŴ the
    unrounded fp32 sum — exact on integer inputs."""
    torch = require_cuda()
    (X, W, dY), (O, dI, dW) = _layer(ax, m, k, n, transposed, "int", torch.bfloat16,
                                     grad_f32=True)
    rO, rI, rW = fc.fc_layer(X, W, dY)
    for got, ref in ((O, rO), (dI, rI)):
        assert np.array_equal(bf16_bits_of(got), synthdata.bf16_bits(synthdata.bf16_round(ref)))
    assert dW.dtype == torch.float32
    np.testing.assert_array_equal(to_host_f64(dW), rW)


def test_grad_f32_random_beats_bf16_rounding(ax):
    torch = require_cuda()
    m, k, n = 2048, 1024, 768
    (X, W, dY), (O, dI, dW) = _layer(ax, m, k, n, False, "uniform", torch.bfloat16,
                                     grad_f32=True)
    rW = fc.fc_backward_weight(X, dY)
    absW = fc.fc_backward_weight(np.abs(X), np.abs(dY))
    u = 2.0 ** -24
    assert np.all(np.abs(to_host_f64(dW) - rW) <= m * u / (1 - m * u) * absW)


def test_zero_tokens(ax):
    """m = 0 (an empty batch): O and dI are empty, dŴ = Xᵀ dY over no rows = 0."""
    torch = require_cuda()
    k, n = 256, 136
    h = ax.axonn_fc_create(0, k, n)
    W = torch.ones(k * n, dtype=torch.bfloat16, device="cuda")
    I = torch.empty((0, k), dtype=torch.bfloat16, device="cuda")
    dO = torch.empty((0, n), dtype=torch.bfloat16, device="cuda")
    O = torch.empty((0, n), dtype=torch.bfloat16, device="cuda")
    dI = torch.empty((0, k), dtype=torch.bfloat16, device="cuda")
    dW = torch.full((k * n,), float("nan"), dtype=torch.bfloat16, device="cuda")
    ax.axonn_fc_forward(h, I, W, O)
    ax.axonn_fc_backward(h, dO, dI, dW)
    ax.axonn_grads_sync()
    torch.cuda.synchronize()
    assert torch.count_nonzero(dW).item() == 0 and not torch.isnan(dW).any()
    ax.axonn_fc_destroy(h)


def test_backward_before_forward_is_state_error(ax):
    torch = require_cuda()
    h = ax.axonn_fc_create(128, 128, 128)
    t = torch.zeros((128, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_fc_backward(h, t, t, t)
    assert e.value.status == ax.AXONN_ERR_STATE
    ax.axonn_fc_destroy(h)


def test_kernel_launch_counter_and_profile(ax):
    torch = require_cuda()
    n0 = ax.axonn_kernel_launches()
    ax.axonn_profile_enable(True)
    _layer(ax, 256, 256, 256, False, "uniform", torch.bfloat16)
    ax.axonn_profile_enable(False)
    launches, ms, flops = ax.axonn_profile_read()
    assert ax.axonn_kernel_launches() - n0 == 3 == launches
    assert flops == 3 * 2 * 256 ** 3 and ms > 0


def test_cuda_graph_capture_and_replay(ax):
    """Alg. 1 forward + backward + grads_sync captured in one CUDA graph and
    replayed on fresh inputs gives the oracle's results (integer inputs, exact)."""
    torch = require_cuda()
    m, k, n = 384, 256, 520
    h = ax.axonn_fc_create(m, k, n, False, ax.AXONN_BF16)
    bufs = {name: torch.zeros(shape, dtype=torch.bfloat16, device="cuda") for name, shape in
            (("I", (m, k)), ("W", (k * n,)), ("dO", (m, n)), ("O", (m, n)), ("dI", (m, k)),
             ("dW", (k * n,)))}
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):   # warm-up (first-launch attribute setup happens here)
        ax.axonn_fc_forward(h, bufs["I"], bufs["W"], bufs["O"], s)
        ax.axonn_fc_backward(h, bufs["dO"], bufs["dI"], bufs["dW"], s)
        ax.axonn_grads_sync(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        ax.axonn_fc_forward(h, bufs["I"], bufs["W"], bufs["O"], s)
        ax.axonn_fc_backward(h, bufs["dO"], bufs["dI"], bufs["dW"], s)
        ax.axonn_grads_sync(s)
    for seed in (5, 6):
        X, W, dY = synthdata.layer_tensors(m, k, n, seed, kind="int")
        bufs["I"].copy_(to_dev(X, torch.bfloat16))
        bufs["W"].copy_(to_dev(W, torch.bfloat16).reshape(-1))
        bufs["dO"].copy_(to_dev(dY, torch.bfloat16))
        g.replay()
        torch.cuda.synchronize()
        for got, ref in zip((bufs["O"], bufs["dI"], bufs["dW"].reshape(k, n)), fc.fc_layer(X, W, dY)):
            assert np.array_equal(bf16_bits_of(got), synthdata.bf16_bits(synthdata.bf16_round(ref)))
    ax.axonn_fc_destroy(h)


def test_bf16_shards_need_16_byte_rows(ax):
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_fc_create(64, 60, 64)
    assert e.value.status == ax.AXONN_ERR_SHAPE and "multiples of 8" in str(e.value)
    h = ax.axonn_fc_create(64, 60, 64, False, ax.AXONN_F32)   # fp32 test mode: no TMA
    ax.axonn_fc_destroy(h)


@pytest.mark.parametrize("m", [1, 127, 129, 1000])
def test_ragged_token_counts(ax, m):
    """m_l is unrestricted: a single token and counts that are not tile multiples."""
    torch = require_cuda()
    (X, W, dY), outs = _layer(ax, m, 136, 264, False, "int", torch.bfloat16)
    for got, ref in zip(outs, fc.fc_layer(X, W, dY)):
        assert np.array_equal(bf16_bits_of(got), synthdata.bf16_bits(synthdata.bf16_round(ref)))


@pytest.mark.parametrize("m,k,n", [(256, 512, 1024), (384, 200, 136)])
def test_gelu_layer_g1(ax, m, k, n):
    """fc1's GeLU through the ABI at G = 1 (reading R18): O = GELU(X W) and the
    backward on dZ = dY ⊙ GELU'(X W), against oracle.act; the activation pass
    itself against GELU of the GPU's own Z within one bf16 ulp."""
    torch = require_cuda()
    from oracle import act
    X, W, dY = synthdata.layer_tensors(m, k, n, 4, kind="uniform")
    h = ax.axonn_fc_create(m, k, n, False, ax.AXONN_BF16, 1, ax.AXONN_ACT_GELU)
    I, What, dO = to_dev(X, torch.bfloat16), to_dev(W.reshape(1, -1), torch.bfloat16).reshape(-1), \
        to_dev(dY, torch.bfloat16)
    O = empty_dev(m, n, torch.bfloat16)
    dI = empty_dev(m, k, torch.bfloat16)
    dW = empty_dev(1, k * n, torch.bfloat16).reshape(-1)
    ax.axonn_fc_forward(h, I, What, O)
    ax.axonn_fc_backward(h, dO, dI, dW)
    ax.axonn_grads_sync()
    torch.cuda.synchronize()
    ax.axonn_fc_destroy(h)
    Z = fc.fc_forward(X, W)
    dZ = dY * act.gelu_grad(Z)
    for name, got, ref in (("O", O, act.gelu(Z)), ("dI", dI, fc.fc_backward_input(dZ, W)),
                           ("dW", dW.reshape(k, n), fc.fc_backward_weight(X, dZ))):
        e = normwise_err(to_host_f64(got), ref)
        assert e <= 2e-2, (name, e)


def test_gelu_activation_pass_g1(ax):
    """The activation pass itself: on integer inputs Z = X W is exact and
    bf16(Z) is the same on both sides, so O must be bf16(GELU(bf16(Z))) up to
    one bf16 ulp plus the fp32 cancellation of 1 + erf(x/√2) for x < 0
    (absolute |x|·2^-22)."""
    torch = require_cuda()
    from oracle import act
    m, k, n = 256, 64, 512
    X, W, dY = synthdata.layer_tensors(m, k, n, 5, kind="int")
    X = X / 4.0            # Z in [-64, 64]: the whole GeLU range is exercised
    h = ax.axonn_fc_create(m, k, n, False, ax.AXONN_BF16, 1, ax.AXONN_ACT_GELU)
    I, What, dO = to_dev(X, torch.bfloat16), to_dev(W.reshape(1, -1), torch.bfloat16).reshape(-1), \
        to_dev(dY, torch.bfloat16)
    O = empty_dev(m, n, torch.bfloat16)
    dI = empty_dev(m, k, torch.bfloat16)
    dW = empty_dev(1, k * n, torch.bfloat16).reshape(-1)
    ax.axonn_fc_forward(h, I, What, O)
    ax.axonn_fc_backward(h, dO, dI, dW)
    torch.cuda.synchronize()
    ax.axonn_fc_destroy(h)
    Zb = synthdata.bf16_round(fc.fc_forward(X, W)).astype(np.float64)
    want = act.gelu(Zb)
    got = to_host_f64(O)
    tol = np.abs(want) * 2.0 ** -7 + np.abs(Zb) * 2.0 ** -22
    assert np.all(np.abs(got - want) <= tol), np.max(np.abs(got - want) - tol)


def test_gelu_mlp_chain_g1(ax):
    """fc1 (GeLU) -> fc2 chained on device at G = 1 vs oracle.act.mlp."""
    torch = require_cuda()
    from oracle import act
    m, h = 256, 128
    X = synthdata.tensor((m, h), 31)
    W1 = synthdata.bf16_round(synthdata.tensor((h, 4 * h), 32) * 0.1)
    W2 = synthdata.bf16_round(synthdata.tensor((4 * h, h), 33) * 0.05)
    dY = synthdata.tensor((m, h), 34)
    h1 = ax.axonn_fc_create(m, h, 4 * h, False, ax.AXONN_BF16, 1, ax.AXONN_ACT_GELU)
    h2 = ax.axonn_fc_create(m, 4 * h, h, True, ax.AXONN_BF16)
    dev = lambda a: to_dev(a, torch.bfloat16)  # noqa: E731
    Xd, W1d, W2d, dYd = dev(X), dev(W1.reshape(1, -1)).reshape(-1), dev(W2.reshape(1, -1)).reshape(-1), dev(dY)
    A = empty_dev(m, 4 * h, torch.bfloat16)
    O = empty_dev(m, h, torch.bfloat16)
    dA = empty_dev(m, 4 * h, torch.bfloat16)
    dX = empty_dev(m, h, torch.bfloat16)
    dW1 = empty_dev(1, h * 4 * h, torch.bfloat16).reshape(-1)
    dW2 = empty_dev(1, h * 4 * h, torch.bfloat16).reshape(-1)
    ax.axonn_fc_forward(h1, Xd, W1d, A)
    ax.axonn_fc_forward(h2, A, W2d, O)
    ax.axonn_fc_backward(h2, dYd, dA, dW2)
    ax.axonn_fc_backward(h1, dA, dX, dW1)
    ax.axonn_grads_sync()
    torch.cuda.synchronize()
    for hh in (h1, h2):
        ax.axonn_fc_destroy(hh)
    r = act.mlp(X, W1, W2, dY)
    for name, got, ref in (("O", O, r["O"]), ("dX", dX, r["dX"]), ("dW1", dW1.reshape(h, 4 * h), r["dW1"]),
                           ("dW2", dW2.reshape(4 * h, h), r["dW2"])):
        e = normwise_err(to_host_f64(got), ref)
        assert e <= 2e-2, (name, e)
