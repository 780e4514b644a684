"""The stream-K tail's decomposition (gemm_tc.cu SkParams), checked on the host
through axonn_stream_k_items, which runs the kernel's own item functions: the
split tiles' K-blocks are covered exactly once, every tile is whole or one
HEAD + one TAIL on consecutive CTA pairs, each pair does its HEAD first and its
TAIL last (what makes the claim protocol wait only on pairs that have
started), and the pairs' shares differ by at most one K-block."""
import pytest

import paper_2502_08145_b200 as ax

# (sk_tiles, K-blocks per tile, CTA pairs): the C2 launches that take the tail
# on a 148-SM B200 (qkv dW 384 tiles -> 384 % 74 + 74 = 88; proj dW 128), the
# 256x256 tiles of AXONN_PAIR_MT=1 (256 tiles -> 34 + 74), ragged K, the
# smallest and largest split (pairs, 2 * pairs - 1) and a small grid.
CASES = [(88, 256, 74), (128, 256, 74), (108, 64, 74), (136, 18, 74), (74, 16, 74),
         (147, 17, 74), (5, 33, 3), (7, 100, 4)]


def items(sk_tiles, kb, pairs):
    return [ax.axonn_stream_k_items(sk_tiles, kb, p, pairs) for p in range(pairs)]


@pytest.mark.parametrize("sk_tiles,kb,pairs", CASES)
def test_every_k_block_once_and_pieces_pair_up(sk_tiles, kb, pairs):
    per_pair = items(sk_tiles, kb, pairs)
    cover = {}
    pieces = {}
    for p, its in enumerate(per_pair):
        for tile, role, k0, k1 in its:
            assert 0 <= tile < sk_tiles and 0 <= k0 < k1 <= kb
            for u in range(k0, k1):
                assert (tile, u) not in cover, f"K-block {u} of tile {tile} twice"
                cover[(tile, u)] = p
            pieces.setdefault(tile, []).append((p, role, k0, k1))
    assert len(cover) == sk_tiles * kb
    for tile, ps in pieces.items():
        if len(ps) == 1:
            assert ps[0][1] == 0 and (ps[0][2], ps[0][3]) == (0, kb)
        else:
            assert len(ps) == 2, f"tile {tile} in {len(ps)} pieces"
            (pa, ra, a0, a1), (pb, rb, b0, b1) = sorted(ps)
            # the HEAD [0, h) on pair p, the TAIL [h, kb) on pair p + 1
            assert (ra, rb) == (1, 2) and pb == pa + 1
            assert a0 == 0 and a1 == b0 and b1 == kb and 0 < a1 < kb


@pytest.mark.parametrize("sk_tiles,kb,pairs", CASES)
def test_head_first_tail_last_and_balanced(sk_tiles, kb, pairs):
    per_pair = items(sk_tiles, kb, pairs)
    units = sk_tiles * kb
    for p, its in enumerate(per_pair):
        roles = [r for _, r, _, _ in its]
        assert roles.count(1) <= 1 and roles.count(2) <= 1
        if 1 in roles:
            assert roles[0] == 1, "a HEAD must be the pair's first item"
        if 2 in roles:
            assert roles[-1] == 2, "a TAIL must be the pair's last item"
        share = sum(k1 - k0 for _, _, k0, k1 in its)
        assert share in (units // pairs, -(-units // pairs))
        assert share >= kb  # at least one tile's worth: no tile has three pieces


def test_arguments():
    with pytest.raises(ax.AxonnError) as e:
        ax.axonn_stream_k_items(10, 16, 0, 74)   # fewer split tiles than pairs
    assert e.value.status == ax.AXONN_ERR_ARG
    with pytest.raises(ax.AxonnError):
        ax.axonn_stream_k_items(100, 16, 74, 74)  # pair out of range
