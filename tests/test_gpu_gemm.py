"""Parity of the three local products (Alg. 1 lines 3, 11, 13) through the C ABI
(axonn_gemm) against the fp64 oracle (oracle.fc).

  * integer inputs in [-4, 4]: every partial sum is an exact integer < 2^24, so
    the tcgen05 result must equal RNE_bf16(exact) bit for bit — catches any
    tile, swizzle, descriptor or indexing bug;
  * uniform(-1,1) bf16 inputs: normwise error <= 2e-2 (BASELINE.json
    north_star);
  * fp32 test mode (SIMT): bit-exact on integers, <= 1e-5 on random inputs.
Shapes span several 128x256 tiles, ragged tails in M, N and K, strided rows and
the degenerate K == 0 and M == 0 cases."""
import numpy as np
import pytest

import synthdata
from oracle import fc
from gpu_util import (bf16_bits_of, empty_dev, normwise_err, require_cuda, round_up, to_dev,
                      to_host_f64)

pytestmark = pytest.mark.gpu

OPS = {"NN": 0, "NT": 1, "TN": 2}


def _operands(op, M, N, K, kind, seed=42):
    # storage layouts of A and B for each op (include/axonn.h)
    a_shape = (K, M) if op == "TN" else (M, K)
    b_shape = (N, K) if op == "NT" else (K, N)
    A = synthdata.tensor(a_shape, 1000 + M, seed, kind)
    B = synthdata.tensor(b_shape, 2000 + N, seed, kind)
    return A, B


def _oracle(op, A, B):
    if op == "NN":
        return fc.fc_forward(A, B)             # I x W
    if op == "NT":
        return fc.fc_backward_input(A, B)      # dO x W^T
    return fc.fc_backward_weight(A, B)         # I^T x dO


def _run(op, A, B, M, N, dtype, pad=0, out_f32=False, ldc=None):
    """out_f32: bf16 operands, fp32 C (AXONN_BF16_GRADF32, the dW product of
    fp32 gradient reduction)."""
    torch = require_cuda()
    import paper_2502_08145_b200 as ax
    lda = round_up(A.shape[1]) + pad
    ldb = round_up(B.shape[1]) + pad
    ldc = (round_up(N) + pad) if ldc is None else ldc
    dA = to_dev(A, dtype, lda)
    dB = to_dev(B, dtype, ldb)
    cdt = torch.float32 if out_f32 else dtype
    # output inside a NaN canary: 40 extra rows and the ld padding must stay NaN
    # (compute-sanitizer is closed on this pool; this is our out-of-bounds check)
    guard = torch.full((M + 40, max(ldc, 1)), float("nan"), dtype=cdt, device="cuda")
    dC = guard[:M, :N]
    K = A.shape[0] if op == "TN" else A.shape[1]
    code = (ax.AXONN_BF16_GRADF32 if out_f32 else
            ax.AXONN_F32 if dtype == torch.float32 else ax.AXONN_BF16)
    ax.axonn_gemm(OPS[op], code, M, N, K, dA, lda, dB, ldb, dC, ldc)
    torch.cuda.synchronize()
    assert torch.isnan(guard[M:, :].float()).all(), "write below the last row"
    if ldc > N:
        assert torch.isnan(guard[:, N:].float()).all(), "write past the last column"
    return dC


SHAPES = [(128, 256, 64), (256, 512, 128), (384, 768, 320), (300, 520, 200), (257, 129, 65),
          (1, 8, 8), (129, 257, 1000), (1024, 1024, 1024), (640, 2304, 96)]


@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_bf16_integer_bit_exact(op, M, N, K):
    torch = require_cuda()
    A, B = _operands(op, M, N, K, "int")
    ref = _oracle(op, A, B)
    want = synthdata.bf16_bits(synthdata.bf16_round(ref))
    got = bf16_bits_of(_run(op, A, B, M, N, torch.bfloat16))
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} mismatches, first at {bad[:3].tolist()}"


# Launches whose tiles leave the last wave of CTA pairs partly idle take the
# stream-K tail (gemm_tc.cu SkParams): on a 148-SM B200, 4096 x 4096 is 128
# tiles of 512x256 (1.73 waves of 74 pairs; 256 tiles of 256x256 with
# AXONN_PAIR_MT=1), 4000 x 4100 x 1100 is 136 ragged tiles with a ragged K.
SK_SHAPES = [(4096, 4096, 1024), (4000, 4100, 1100)]


def _expect_stream_k():
    import os
    torch = require_cuda()
    return (torch.cuda.get_device_properties(0).multi_processor_count == 148
            and os.environ.get("AXONN_SK", "1") != "0"
            and os.environ.get("AXONN_SCHED") != "static"
            and os.environ.get("AXONN_GEMM_VARIANT") != "single")


@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("M,N,K", SK_SHAPES)
def test_stream_k_tail_integer_bit_exact(op, M, N, K):
    """The contributor's fp32 partial sums (K-blocks [0, t0)) plus the
    finisher's rest reach the exact integer sums: bit-exact after RNE."""
    torch = require_cuda()
    import paper_2502_08145_b200 as ax
    A, B = _operands(op, M, N, K, "int")
    want = synthdata.bf16_bits(synthdata.bf16_round(_oracle(op, A, B)))
    n0 = ax.axonn_stream_k_launches()
    got = bf16_bits_of(_run(op, A, B, M, N, torch.bfloat16))
    if _expect_stream_k():
        assert ax.axonn_stream_k_launches() == n0 + 1, "the stream-K tail did not run"
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} mismatches, first at {bad[:3].tolist()}"


@pytest.mark.parametrize("M,N,K", SK_SHAPES)
def test_stream_k_tail_deterministic_and_fp32_output(M, N, K):
    """Fixed split points and addition order: the same launch twice is
    bit-identical on random inputs; the fp32-output dW product is exact on
    integers."""
    torch = require_cuda()
    A, B = _operands("TN", M, N, K, "uniform")
    c1 = bf16_bits_of(_run("TN", A, B, M, N, torch.bfloat16))
    c2 = bf16_bits_of(_run("TN", A, B, M, N, torch.bfloat16))
    assert np.array_equal(c1, c2)
    A, B = _operands("TN", M, N, K, "int")
    got = to_host_f64(_run("TN", A, B, M, N, torch.bfloat16, out_f32=True))
    np.testing.assert_array_equal(got, _oracle("TN", A, B))


@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("M,N,K", [(384, 768, 320), (300, 520, 200), (2048, 1536, 1024),
                                   (4000, 4100, 1100)])
def test_bf16_random_within_tolerance(op, M, N, K):
    torch = require_cuda()
    A, B = _operands(op, M, N, K, "uniform")
    ref = _oracle(op, A, B)
    got = to_host_f64(_run(op, A, B, M, N, torch.bfloat16, pad=8))
    assert normwise_err(got, ref) <= 2e-2
    # one bf16 rounding of an fp32 sum: per element within 2^-8 relative + accumulation slack
    assert np.all(np.abs(got - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-5 * np.sqrt(K))


@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("M,N,K", [(300, 520, 200), (257, 129, 65), (64, 64, 1)])
def test_f32_mode(op, M, N, K):
    torch = require_cuda()
    A, B = _operands(op, M, N, K, "int")
    got = to_host_f64(_run(op, A, B, M, N, torch.float32))
    np.testing.assert_array_equal(got, _oracle(op, A, B))
    A, B = _operands(op, M, N, K, "uniform")
    ref = _oracle(op, A, B)
    assert normwise_err(to_host_f64(_run(op, A, B, M, N, torch.float32)), ref) <= 1e-5


# ---- fp32 output of the dW product (AXONN_BF16_GRADF32, reading R17) ----
@pytest.mark.parametrize("M,N,K", SHAPES + [(256, 132, 512), (512, 260, 96)])
def test_tn_fp32_output_integer_bit_exact(M, N, K):
    """The unrounded fp32 accumulator: exact integers (|sum| <= 16 K < 2^24)."""
    torch = require_cuda()
    A, B = _operands("TN", M, N, K, "int")
    got = to_host_f64(_run("TN", A, B, M, N, torch.bfloat16, out_f32=True))
    np.testing.assert_array_equal(got, _oracle("TN", A, B))


@pytest.mark.parametrize("M,N,K,ldc", [(384, 768, 320, None), (300, 520, 200, 524),
                                       (257, 129, 65, 129), (2048, 1536, 1024, None)])
def test_tn_fp32_output_random_within_gamma_bound(M, N, K, ldc):
    """fp32 accumulation of exact bf16 products in any order: |got - ref| <=
    gamma_K * sum|a||b| with gamma_K = K u / (1 - K u), u = 2^-24 (the
    standard dot-product bound).  ldc 524 = padded rows (per-thread vector
    stores), 129 = odd rows (scalar stores); None = TMA-store epilogue."""
    torch = require_cuda()
    A, B = _operands("TN", M, N, K, "uniform")
    ref = _oracle("TN", A, B)
    absref = _oracle("TN", np.abs(A), np.abs(B))
    got = to_host_f64(_run("TN", A, B, M, N, torch.bfloat16, out_f32=True, ldc=ldc))
    u = 2.0 ** -24
    gamma = K * u / (1 - K * u)
    assert np.all(np.abs(got - ref) <= gamma * absref)
    # and strictly better than the bf16-output product
    assert normwise_err(got, ref) <= 1e-5


def test_tn_fp32_output_full_size_sampled():
    """BASELINE.json C2 fc2 dW shape (M=4h, N=h, K=16384 tokens) in fp32."""
    torch = require_cuda()
    M, N, K = 16384, 4096, 16384
    A, B = _operands("TN", M, N, K, "uniform")
    C = _run("TN", A, B, M, N, torch.bfloat16, out_f32=True)
    rng = np.random.default_rng(0)
    rows = rng.integers(0, M, 4096)
    cols = rng.integers(0, N, 4096)
    ref = fc.dot_entries(A.T, B, rows, cols)
    absref = fc.dot_entries(np.abs(A.T), np.abs(B), rows, cols)
    got = C[torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()].double().cpu().numpy()
    u = 2.0 ** -24
    assert np.all(np.abs(got - ref) <= K * u / (1 - K * u) * absref)


@pytest.mark.parametrize("op", [0, 1])
def test_fp32_output_only_for_tn(op):
    torch = require_cuda()
    import paper_2502_08145_b200 as ax
    A = torch.zeros((64, 64), dtype=torch.bfloat16, device="cuda")
    C = torch.zeros((64, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_gemm(op, ax.AXONN_BF16_GRADF32, 64, 64, 64, A, 64, A, 64, C, 64)
    assert e.value.status == ax.AXONN_ERR_ARG and "TN" in str(e.value)


@pytest.mark.parametrize("op", list(OPS))
def test_k_zero_writes_zeros_and_m_zero_is_noop(op):
    torch = require_cuda()
    import paper_2502_08145_b200 as ax
    C = torch.full((16, 24), 7.0, dtype=torch.bfloat16, device="cuda")
    A = torch.zeros((16, 8), dtype=torch.bfloat16, device="cuda")
    ax.axonn_gemm(OPS[op], ax.AXONN_BF16, 16, 24, 0, A, 8, A, 8, C, 24)
    torch.cuda.synchronize()
    assert torch.count_nonzero(C).item() == 0
    ax.axonn_gemm(OPS[op], ax.AXONN_BF16, 0, 24, 8, A, 8, A, 24, C, 24)


def test_deterministic():
    torch = require_cuda()
    A, B = _operands("TN", 1024, 1024, 2048, "uniform")
    c1 = bf16_bits_of(_run("TN", A, B, 1024, 1024, torch.bfloat16))
    c2 = bf16_bits_of(_run("TN", A, B, 1024, 1024, torch.bfloat16))
    assert np.array_equal(c1, c2)


def test_bad_alignment_is_an_error():
    torch = require_cuda()
    import paper_2502_08145_b200 as ax
    A = torch.zeros((64, 66), dtype=torch.bfloat16, device="cuda")
    C = torch.zeros((64, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_gemm(0, ax.AXONN_BF16, 64, 64, 60, A, 66, A, 66, C, 64)
    assert e.value.status == ax.AXONN_ERR_ARG


@pytest.mark.parametrize("op,M,N,K", [("NN", 16384, 12288, 4096),   # C2 QKV forward
                                      ("NT", 16384, 4096, 16384),   # C2 fc2 backward dI
                                      ("TN", 16384, 4096, 16384)])  # C2 fc2 dW (M=4h rows)
def test_full_size_sampled(op, M, N, K):
    """BASELINE.json C2 shapes in the launch configuration bench.py times; 4096
    sampled entries each checked against an exact fp64 dot product."""
    torch = require_cuda()
    A, B = _operands(op, M, N, K, "uniform")
    C = _run(op, A, B, M, N, torch.bfloat16)
    rng = np.random.default_rng(0)
    rows = rng.integers(0, M, 4096)
    cols = rng.integers(0, N, 4096)
    AA = A.T if op == "TN" else A
    BB = B.T if op == "NT" else B
    ref = fc.dot_entries(AA, BB, rows, cols)
    got = C[torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()].double().cpu().numpy()
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 2e-2
    assert np.all(np.abs(got - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-5 * np.sqrt(K))


@pytest.mark.parametrize("env", [{"AXONN_GEMM_VARIANT": "single"}, {"AXONN_PAIR_MT": "1"},
                                 {"AXONN_GROUP_M": "-8"}, {"AXONN_SCHED": "static"},
                                 {"AXONN_SPLIT_RELEASE": "0"}, {"AXONN_SK": "0"},
                                 {"AXONN_MT2_DEEP": "0"}, {"AXONN_PDL": "0"}])
def test_alternative_kernel_configurations(env):
    """The 1-CTA kernel, the 256x256 CTA-pair tile, the transposed raster,
    static tile scheduling, whole-tile accumulator release, no stream-K tail,
    the 3-stage 512x256 pipeline and plain stream order instead of the
    programmatic dependent launch (selected by
    environment, read once per process) pass the same bit-exact integer and
    full-size checks."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(here, "test_gpu_gemm.py"), "-k",
                        "integer or full_size or random or stream_k"],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
