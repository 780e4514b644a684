"""The multi-GPU path's choice of fused reduction mode (sym.cu fused_mode,
through axonn_fused_mode: the same call axonn_fc_create makes), on the host:
the defaults for the shapes the bench runs, every switch, and the cases that
stay unfused (NCCL)."""
import os

import pytest

import paper_2502_08145_b200 as ax

SWITCHES = ("AXONN_REDPAIR", "AXONN_RED_MIN_K", "AXONN_EXCHANGE", "AXONN_XSUM", "AXONN_PAIRSUM")


@pytest.fixture
def env():
    saved = {k: os.environ.get(k) for k in SWITCHES}
    for k in SWITCHES:
        os.environ.pop(k, None)
    yield os.environ
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def test_defaults_on_the_c3_proxy_layers(env):
    # 20B block on (2,2,1,1), m = 8192 (bench.py N=4): the forward AR of QKV
    # (K = 3584) and fc2 (K = 14336), the backward AR of QKV (K = 10752)
    assert ax.axonn_fused_mode(2, 2, 8192, 10752, 3584) == "red_add_pair"
    assert ax.axonn_fused_mode(2, 2, 8192, 3584, 14336) == "multimem_red"
    assert ax.axonn_fused_mode(2, 2, 8192, 3584, 10752) == "multimem_red"
    assert ax.axonn_fused_mode(2, 2, 8192, 3584, 8191) == "red_add_pair"   # the threshold
    assert ax.axonn_fused_mode(2, 2, 8192, 3584, 8192) == "multimem_red"
    # wider axes: scatter + owner phase; fp32 (AXONN_BF16_GRADF32 gradients):
    # no red.add path, the exchange on 2 ranks
    assert ax.axonn_fused_mode(4, 2, 8192, 3584, 3584) == "scatter"
    assert ax.axonn_fused_mode(8, 2, 64, 64, 64) == "scatter"
    assert ax.axonn_fused_mode(2, 4, 3584, 3584, 8192) == "exchange"
    assert ax.axonn_fused_mode(4, 4, 3584, 3584, 8192) == "scatter"


def test_unfused_cases(env):
    assert ax.axonn_fused_mode(1, 2, 64, 64, 64) == "none"    # no reduction
    assert ax.axonn_fused_mode(2, 2, 0, 64, 64) == "none"     # empty output
    assert ax.axonn_fused_mode(2, 2, 64, 64, 0) == "none"     # K = 0: zeros, nothing to reduce
    assert ax.axonn_fused_mode(2, 2, 64, 12, 64) == "none"    # rows not whole 16-B units
    assert ax.axonn_fused_mode(2, 4, 64, 6, 64) == "none"
    assert ax.axonn_fused_mode(3, 2, 8, 16, 8) == "none"      # 128 elements over 3 owners


def test_switches(env):
    env["AXONN_REDPAIR"] = "0"
    assert ax.axonn_fused_mode(2, 2, 8192, 10752, 3584) == "exchange"
    env["AXONN_EXCHANGE"] = "0"
    assert ax.axonn_fused_mode(2, 2, 8192, 10752, 3584) == "scatter"
    env["AXONN_REDPAIR"] = "1"
    assert ax.axonn_fused_mode(2, 2, 8192, 3584, 14336) == "red_add_pair"  # at every K
    env["AXONN_REDPAIR"] = "2"
    env["AXONN_RED_MIN_K"] = "0"
    assert ax.axonn_fused_mode(2, 2, 8192, 10752, 3584) == "multimem_red"
    env["AXONN_XSUM"] = "1"
    assert ax.axonn_fused_mode(2, 2, 8192, 10752, 3584) == "xsum"
    env["AXONN_PAIRSUM"] = "1"
    assert ax.axonn_fused_mode(2, 2, 8192, 10752, 3584) == "pair_sum"
    # none of the 2-rank bf16 modes touch wider axes or fp32 (fp32 2-rank:
    # scatter here, AXONN_EXCHANGE=0 is still set; the exchange otherwise)
    assert ax.axonn_fused_mode(4, 2, 8192, 3584, 3584) == "scatter"
    assert ax.axonn_fused_mode(2, 4, 3584, 3584, 8192) == "scatter"
    env["AXONN_EXCHANGE"] = "1"
    assert ax.axonn_fused_mode(2, 4, 3584, 3584, 8192) == "exchange"


def test_arguments():
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_fused_mode(0, 2, 8, 8, 8)
    assert e.value.status == ax.AXONN_ERR_ARG
    with pytest.raises(ax.AxonnError):
        ax.axonn_fused_mode(2, 3, 8, 8, 8)
