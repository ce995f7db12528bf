"""The library's traffic model (paper_2105_14450_b200/traffic.py) against the reference's
cost model (oracle port of traffic::, pinned to the reference's golden costs in
test_oracle_golden.py): on a p-cube the forward is identical and the backward differs by
exactly the documented reuse terms. The GPU side (tools/mp_parity.py) checks the measured
counters against the same model on 2- and 4-GPU grids. CPU only."""
import pytest

from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import traffic as T


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("cfg", [(2, 8, 2, 16), (4, 36, 6, 72), (32, 512, 16, 1024),
                                 (64, 1024, 16, 2048)])
@pytest.mark.parametrize("flash", [True, False])
def test_cube_traffic_is_reference_minus_documented_reuse(p, cfg, flash):
    b, s, n, h = cfg
    if b % p or s % p or n % p or h % (p * p):
        pytest.skip("indivisible on this cube")
    ref_f, ref_b = O.traffic_layer(b, s, n, h, p)
    ours_f, ours_b = T.layer_traffic(b, s, n, h, (p, p, p), flash=flash)
    dev = T.reference_deviation(b, s, n, h, p, flash=flash)
    assert ours_f == ref_f
    assert ours_b == ref_b - sum(dev.values())
    if p == 1:
        assert ours_f == ours_b == 0


def test_subgrid_traffic_is_positive_and_balanced():
    # 2x1x1 moves only the x-axis weight gathers / gradient scatters and vector traffic;
    # 2x2x1 and 1x2x2 add activation traffic
    b, s, n, h = 4, 512, 16, 1024
    f211, b211 = T.layer_traffic(b, s, n, h, (2, 1, 1))
    assert f211 == 12 * h * h + 2 * (13 * h // 2)  # weights gathered once + 2 vector packs
    for dims in [(2, 2, 1), (1, 2, 2), (2, 1, 2)]:
        f, bw = T.layer_traffic(b, s, n, h, dims)
        assert f > 0 and bw > 0
