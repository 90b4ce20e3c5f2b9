"""Host-side guards of the distributed drivers (no GPU needed)."""

import pytest


def test_global_scaling_refused_on_more_than_one_rank():
    """GLOBAL scaling needs one exponent over the whole operand
    (split.py:131-134); the distributed drivers split per rank, so they refuse
    it instead of returning factors that differ from the reference."""
    import paper_2509_23565_b200 as oz
    from paper_2509_23565_b200.hpl import check_scaling
    from paper_2509_23565_b200.split import ScalingMode
    glob = oz.GemmBackend.int8(7, scaling=ScalingMode.GLOBAL)
    check_scaling(glob, 1)                                  # one rank: the single-GPU path
    check_scaling(oz.GemmBackend.int8(7), 8)
    check_scaling(oz.GemmBackend.native(), 8)
    with pytest.raises(oz.InvalidParamsError):
        check_scaling(glob, 2)
