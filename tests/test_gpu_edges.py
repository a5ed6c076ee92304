"""Edge cases of the step / reset kernels at the C-ABI boundary: empty reset
masks, ragged batch sizes around the warp / CTA / row-padding boundaries,
non-finite and out-of-range commands (the reference clips with np.clip and
freezes non-finite rows, engine.py:411-449 / 487-512)."""

import numpy as np
import pytest
import torch

from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.randomization import DRParameter, Uniform
from paper_2503_09203_b200.vehicles import load_vehicle

pytestmark = pytest.mark.gpu

FIELDS = ("p", "q", "nu", "act", "steps", "episodes", "diverged")
SPEC = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("mass*", "volume*", "damping*")}


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _batch(veh, n, dtype=torch.float32, substeps=2):
    st = E.make_batch(veh, E.SimConfig(batch_size=n, substeps=substeps), master_seed=11,
                      dtype=dtype)
    E.reset_envs(st, np.ones(n, bool), E.spec_sampler(SPEC))
    return st


def _snap(st):
    return {k: getattr(st, k).clone() for k in FIELDS}


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_empty_reset_mask_changes_nothing(dtype):
    st = _batch(load_vehicle("bluerov"), 77, dtype)
    E.step_batch(st, torch.rand((77, 6), device="cuda", dtype=dtype) * 2 - 1)
    before = _snap(st)
    for sampler in (E.default_sampler, E.spec_sampler(SPEC)):
        E.reset_envs(st, np.zeros(77, bool), sampler)
        for k in FIELDS:
            assert torch.equal(getattr(st, k), before[k]), k


@pytest.mark.parametrize("vehicle", ["bluerov", "lauv", "bluerov_heavy"])
@pytest.mark.parametrize("n", [1, 31, 33, 127, 129])
def test_ragged_batches_equal_rows_of_a_larger_batch(vehicle, n):
    """Rows are independent and keyed by env index: a batch of n envs equals the
    first n rows of a 300-env batch bit for bit (same kernels, padded row
    stride, partial warps and CTAs)."""
    veh = load_vehicle(vehicle)
    big, small = _batch(veh, 300), _batch(veh, n)
    g = torch.Generator(device="cuda").manual_seed(5)
    for t in range(4):
        cmd = torch.rand((300, veh.action_dim), device="cuda", generator=g) * 2.4 - 1.2
        E.step_batch(big, cmd)
        E.step_batch(small, cmd[:n].contiguous())
        if t == 1:  # a mid-rollout partial reset of every third row
            m = np.zeros(300, bool)
            m[::3] = True
            E.reset_envs(big, m, E.spec_sampler(SPEC))
            E.reset_envs(small, m[:n], E.spec_sampler(SPEC))
    for k in FIELDS:
        assert torch.equal(getattr(small, k), getattr(big, k)[:n]), k


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_infinite_commands_clip_like_unit_commands(dtype):
    """np.clip(+-inf, -1, 1) = +-1 (engine.py:412): not a divergence."""
    veh = load_vehicle("bluerov")
    a, b = _batch(veh, 64, dtype), _batch(veh, 64, dtype)
    sign = torch.where(torch.arange(64 * 6, device="cuda").reshape(64, 6) % 3 == 0, -1.0, 1.0)
    sign = sign.to(dtype)
    for _ in range(3):
        E.step_batch(a, sign * float("inf"))
        E.step_batch(b, sign * 7.5)
    for k in FIELDS:
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    assert not bool(a.diverged.any())


def test_nan_command_freezes_only_its_row():
    veh = load_vehicle("bluerov")
    a, b = _batch(veh, 96), _batch(veh, 96)
    cmd = torch.rand((96, 6), device="cuda") * 2 - 1
    bad = cmd.clone()
    bad[40, 3] = float("nan")
    before = _snap(a)
    E.step_batch(a, bad)
    E.step_batch(b, cmd)
    assert a.diverged.nonzero().flatten().tolist() == [40]
    keep = torch.ones(96, dtype=torch.bool, device="cuda")
    keep[40] = False
    for k in ("p", "q", "nu", "act"):
        assert torch.equal(getattr(a, k)[keep], getattr(b, k)[keep]), k
        assert torch.equal(getattr(a, k)[40], before[k][40]), k  # frozen at its last finite state
    assert int(a.steps[40]) == int(before["steps"][40]) + 1
    E.step_batch(a, cmd)  # frozen rows stay frozen, their step counter still advances
    assert torch.equal(a.p[40], before["p"][40]) and int(a.steps[40]) == int(before["steps"][40]) + 2
