"""hsv_sum_rows_async: the rank-order combination of all-gathered partials
(distributed.combine_partials) is bitwise the sequential sum over ranks."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_combine_partials_rank_order_bitwise():
    import torch
    from paper_2604_01176_b200.distributed import bind_library_stream, combine_partials
    bind_library_stream()
    rng = np.random.default_rng(4)
    for world, m in ((1, 5), (2, 1820), (3, 77), (8, 3383)):
        host = rng.standard_normal((world, m)) * 10.0 ** rng.integers(-8, 8, size=(world, m))
        g = torch.from_numpy(host).cuda()
        out = combine_partials(g).cpu().numpy()
        ref = host[0].copy()
        for r in range(1, world):
            ref += host[r]
        assert np.array_equal(out, ref)
