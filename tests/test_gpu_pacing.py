"""GPU parity under the host-paced step grid ("grid pacing"): the grid of
step s is sized from the heavy count of step s - 3, so a sudden jump in heavy traces sends the
items past the estimate to the overflow kernel.  These streams force that jump (a NOP prefix,
then the random c3 / c6 op mix on every trace) and must stay bit-exact with the oracle, through
device and host op streams alike."""
import numpy as np
import pytest

from paper_2605_24259_b200 import gen
from parity_util import assert_parity, run_gpu, run_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_24259_b200 import build
    build.build()


def _nop_prefix(ops, steps):
    ops = ops.copy()
    ops[:steps] = np.zeros((), dtype=ops.dtype)
    return ops


@pytest.mark.parametrize("config,device_ops", [(3, True), (3, False), (6, True)])
def test_heavy_jump_overflows_the_paced_grid(config, device_ops):
    cfgs, ops = gen.random_traces(config, seed=77, trace_begin=0, n_traces=6000, T=64, N=1024)
    ops = _nop_prefix(ops, 12)  # steps 0..11: no heavy trace; step 12 on: ~half of them
    g = run_gpu(cfgs, ops, N=1024, device_ops=device_ops)
    o = run_ref(cfgs, ops, N=1024)
    assert_parity(g, o, what=f"pacing jump c{config}")


def test_alternating_heavy_steps():
    """NOP and random steps alternating in blocks of 4 (the estimate is wrong in both directions)."""
    cfgs, ops = gen.random_traces(3, seed=78, trace_begin=0, n_traces=4000, T=80, N=1024)
    ops = ops.copy()
    for s in range(0, 80, 8):
        ops[s:s + 4] = np.zeros((), dtype=ops.dtype)
    g = run_gpu(cfgs, ops, N=1024)
    o = run_ref(cfgs, ops, N=1024)
    assert_parity(g, o, what="pacing alternating")
