"""the capacity sweep as a GPU batch reproduces the paper's
boundary: hard exclusion refuses below R + A usable blocks and
serves with the resident preserved from R + A on; native / no-admit serve at
every size and lose the resident below R + A.  The paper's case is R=60,
A=70 -> flip at 130; random (R, A) pairs flip at R + A."""
import random

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_capacity_sweep_flips_at_R_plus_A():
    from paper_2605_24259_b200.sweep import flip_points, run_sweep
    rng = random.Random(0)
    pairs = [(60, 70)] + [(rng.randint(1, 400), rng.randint(1, 400)) for _ in range(40)]
    cells = run_sweep(pairs)
    flips = flip_points(cells)
    for R, A in pairs:
        assert flips[(R, A, "hard")] == R + A
        assert flips[(R, A, "native")] == R + A
        assert flips[(R, A, "noadmit")] == R + A
    for c in cells:
        if c["policy"] == "hard":
            assert c["resident_kept"]
            assert c["served"] == (c["U"] >= c["R"] + c["A"])
            assert c["refused"] == (not c["served"])
        else:
            assert c["served"] == (c["U"] >= c["A"])
            assert c["resident_kept"] == (c["U"] >= c["R"] + c["A"])
            if c["served"]:
                assert c["resident_leading"] == c["R"] - max(0, c["A"] - (c["U"] - c["R"]))
    assert flips[(60, 70, "hard")] == 130
