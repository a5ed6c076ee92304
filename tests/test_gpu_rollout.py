"""engine.rollout (uuv_rollout_dl, k_rollout): T control steps in one launch with the state in
registers == T step_batch launches, bit for bit (same substep code, same per-env parameters).

Covers the benchmarked cfg2 kernel class, K = 8, mixed fleets, fin vehicles, the generic
layout (rotor nets), frozen/diverging rows, command rings that wrap, the pose trace, and
the device-side command ring (a producer stream raising a ready counter)."""

import numpy as np
import pytest
import torch
from conftest import product_vehicle

from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.randomization import DRParameter, Uniform, preset

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


FIELDS = ("p", "q", "nu", "act", "steps", "diverged", "episodes")


def pair(make):
    a, b = make(), make()
    for k in FIELDS:
        assert torch.equal(getattr(a, k), getattr(b, k))
    return a, b


def same(a, b, where=""):
    for k in FIELDS:
        assert torch.equal(getattr(a, k), getattr(b, k)), (where, k)


def cfg2(n, dtype, substeps=1):
    def make():
        st = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=n, substeps=substeps),
                          master_seed=0, dtype=dtype)
        spec = {k: DRParameter(k, Uniform(0.8, 1.2))
                for k in ("damping*", "mass*", "thrust_coeff*", "volume*")}
        E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=st.device), E.spec_sampler(spec))
        return st
    return make


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("substeps", [1, 8])
def test_rollout_equals_launched_steps_cfg2(dtype, substeps):
    n, T = 4096, 37
    a, b = pair(cfg2(n, dtype, substeps))
    g = torch.Generator(device="cuda").manual_seed(0)
    ring = (torch.rand((T, n, 6), device="cuda", generator=g) * 2.2 - 1.1).to(dtype)
    ring[5, 9, 2] = float("nan")  # env 9 diverges at step 5 and stays frozen
    for t in range(T):
        E.step_batch(a, ring[t])
    E.rollout(b, ring)
    same(a, b)
    assert bool(b.diverged[9]) and int(b.steps[0]) == T


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_rollout_ring_wraps_and_trace(dtype):
    n, S, T, start = 1000, 5, 23, 3
    a, b = pair(cfg2(n, dtype))
    ring = (torch.rand((S, n, 6), device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(1)) * 2 - 1).to(dtype)
    trace = torch.empty((T, 13, n), dtype=dtype, device="cuda")
    want = []
    for t in range(T):
        E.step_batch(a, ring[(start + t) % S])
        want.append(torch.cat([a.p, a.q, a.nu], dim=1).T.clone())
    E.rollout(b, ring, T, start=start, trace=trace)
    same(a, b)
    assert torch.equal(trace, torch.stack(want))
    # held commands (throughput_probe): (N, A) for every step
    E.rollout(b, ring[0], 4)
    for _ in range(4):
        E.step_batch(a, ring[0])
    same(a, b, "held")


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_rollout_fleet_and_generic_layouts(dtype):
    names = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv")
    vehs = [product_vehicle(x) for x in names + ("rotor_relu",)]  # + the generic layout
    counts = [300, 200, 250, 150, 100, 200]
    n = sum(counts)

    def make():
        st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2),
                                master_seed=4, dtype=dtype)
        E.reset_envs(st, np.ones(n, bool), E.spec_sampler(preset("train")))
        return st

    a, b = pair(make)
    T = 15
    ring = (torch.rand((T, n, a.a_max), device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(2)) * 2 - 1).to(dtype)
    for t in range(T):
        E.step_batch(a, ring[t])
    E.rollout(b, ring)
    # the mixed-fleet kernels: the same per-type code compiled into two different kernels may
    # contract multiply-adds differently (as the per-run fleet dispatch), so the bar is the
    # parity tolerance; counters and flags exact
    for k in ("steps", "diverged", "episodes"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    rtol, atol = (1e-5, 1e-6) if dtype == torch.float32 else (1e-12, 1e-14)
    for k in ("p", "q", "nu", "act"):
        x, y = getattr(a, k).double(), getattr(b, k).double()
        scale = x.abs().amax(dim=1)
        if k == "act":
            scale = scale.clamp(min=100.0)
        err = (x - y).abs().amax(dim=1)
        assert bool((err <= rtol * scale + atol).all()), (k, float((err / scale).max()))


def test_rollout_waits_for_the_device_command_ring():
    """A producer stream fills slot t and raises `ready`; the resident rollout consumes the
    slots as they arrive (launched first, it waits on the counter)."""
    n, T = 2048, 12
    a, b = pair(cfg2(n, torch.float32))
    src = torch.rand((T, n, 6), device="cuda") * 2 - 1
    ring = torch.zeros_like(src)
    ready = torch.zeros(1, dtype=torch.int32, device="cuda")
    consumer, producer = torch.cuda.Stream(), torch.cuda.Stream()
    # the producer's kernels are loaded first: under CUDA lazy loading a kernel's first
    # launch waits for the device, i.e. for the waiting rollout (it would give up after 10 s)
    with torch.cuda.stream(producer):
        torch.cuda._sleep(100)
        ring[0].copy_(src[0])
        ready.fill_(0)
        ring[0].zero_()
    torch.cuda.synchronize()
    with torch.cuda.stream(consumer):
        E.rollout(b, ring, T, ready=ready)
    with torch.cuda.stream(producer):
        for t in range(T):
            torch.cuda._sleep(20000)  # the producer is slower than the stepper
            ring[t].copy_(src[t])
            ready.fill_(t + 1)
    torch.cuda.synchronize()
    for t in range(T):
        E.step_batch(a, src[t])
    same(a, b)


def test_rollout_large_batch_build():
    """From 262,144 envs the 168-register rollout build runs (and k_step's 96-register
    build): still bit for bit the launched steps."""
    n, T = 262_144, 6
    a, b = pair(cfg2(n, torch.float32))
    ring = torch.rand((T, n, 6), device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(3)) * 2 - 1
    for t in range(T):
        E.step_batch(a, ring[t])
    E.rollout(b, ring)
    same(a, b)


def test_rollout_argument_errors():
    st = cfg2(64, torch.float32)()
    with pytest.raises(E.EngineError, match="commands"):
        E.rollout(st, torch.zeros((3, 64, 5), device="cuda"))
    with pytest.raises(E.EngineError, match="commands"):
        E.rollout(st, np.zeros((3, 64, 6)))
    with pytest.raises(E.EngineError, match="trace"):
        E.rollout(st, torch.zeros((3, 64, 6), device="cuda"),
                  trace=torch.zeros((2, 13, 64), device="cuda"))
    E.rollout(st, torch.zeros((3, 64, 6), device="cuda"), 0)  # zero steps: no-op
    assert int(st.steps[0]) == 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_rollout_trace_with_act_rows(dtype):
    """A (T, 13 + A, N) trace also receives act after every step."""
    n, T = 1500, 9
    a, b = pair(cfg2(n, dtype, substeps=2))
    ring = (torch.rand((T, n, 6), device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(5)) * 2 - 1).to(dtype)
    trace = torch.full((T, 19, n), float("nan"), dtype=dtype, device="cuda")
    want = []
    for t in range(T):
        E.step_batch(a, ring[t])
        want.append(torch.cat([a.p, a.q, a.nu, a.act], dim=1).T.clone())
    E.rollout(b, ring, trace=trace)
    same(a, b)
    assert torch.equal(trace, torch.stack(want))


def test_rollout_host_to_host_equals_device_rollout():
    """Pinned host commands and a pinned host trace (13 + A rows): the kernel reads the
    command rows and writes the trace over the host link -- same bits as the device
    rollout and as the launched steps; the call returns with the trace in host memory."""
    n, S, T = 4096, 7, 20
    a, b = pair(cfg2(n, torch.float32))
    c = cfg2(n, torch.float32)()
    ring = torch.rand((S, n, 6), device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(6)) * 2 - 1
    host_ring = ring.cpu().pin_memory()
    host_trace = torch.full((T, 19, n), float("nan")).pin_memory()
    dev_trace = torch.empty((T, 19, n), device="cuda")
    want = []
    for t in range(T):
        E.step_batch(a, ring[(2 + t) % S])
        want.append(torch.cat([a.p, a.q, a.nu, a.act], dim=1).T.cpu())
    res = E.HostStepOut(b)
    E.rollout(b, host_ring, T, start=2, trace=host_trace, out=res)
    E.rollout(c, ring, T, start=2, trace=dev_trace)
    same(a, b)
    same(a, c)
    # out=HostStepOut: the result after the last step, in host memory on return
    assert torch.equal(res.pose, torch.cat([a.p, a.q, a.nu], dim=1).T.cpu())
    assert torch.equal(res.act, a.act.cpu())
    assert torch.equal(res.steps, a.steps.cpu()) and torch.equal(res.diverged, a.diverged.cpu())
    assert torch.equal(host_trace, torch.stack(want))
    assert torch.equal(host_trace, dev_trace.cpu())
    # host commands with a device trace, and device commands with a 13-row host trace
    d = cfg2(n, torch.float32)()
    E.rollout(d, host_ring, T, start=2, trace=dev_trace)
    same(a, d)
    pose = torch.empty((T, 13, n)).pin_memory()
    e = cfg2(n, torch.float32)()
    E.rollout(e, ring, T, start=2, trace=pose)
    same(a, e)
    assert torch.equal(pose, host_trace[:, :13])


def test_rollout_host_argument_errors():
    st = cfg2(64, torch.float32)()
    with pytest.raises(E.EngineError, match="out"):
        E.rollout(st, torch.zeros((3, 64, 6), device="cuda"), out=object())
    other = cfg2(65, torch.float32)()
    with pytest.raises(E.EngineError, match="out: buffers for 65"):
        E.rollout(st, torch.zeros((3, 64, 6), device="cuda"),
                  out=E.HostStepOut(other, fields=("steps",)))
    with pytest.raises(E.EngineError, match="pinned"):
        E.rollout(st, torch.zeros((3, 64, 6)))  # pageable host commands
    with pytest.raises(E.EngineError, match="pinned"):
        E.rollout(st, torch.zeros((3, 64, 6)).pin_memory().double())
    with pytest.raises(E.EngineError, match="trace"):
        E.rollout(st, torch.zeros((3, 64, 6), device="cuda"), trace=torch.zeros((3, 13, 64)))
    with pytest.raises(E.EngineError, match="trace"):
        E.rollout(st, torch.zeros((3, 64, 6), device="cuda"),
                  trace=torch.zeros((3, 15, 64)).pin_memory())
    assert int(st.steps[0]) == 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_rollout_host_buffers_fleet(dtype):
    """Mixed fleet (the generic-fleet kernel), both dtypes: host commands and a host trace
    (13 + a_max rows) give the same bits as device commands and a device trace."""
    names = ("bluerov", "lauv", "hauv")
    vehs = [product_vehicle(x) for x in names]
    counts = [300, 250, 200]
    n, T = sum(counts), 9

    def make():
        st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2),
                                master_seed=6, dtype=dtype)
        E.reset_envs(st, np.ones(n, bool), E.spec_sampler(preset("train")))
        return st

    a, b = pair(make)
    w = a.a_max
    ring = (torch.rand((T, n, w), device="cuda", generator=torch.Generator(
        device="cuda").manual_seed(8)) * 2 - 1).to(dtype)
    dev_trace = torch.empty((T, 13 + w, n), dtype=dtype, device="cuda")
    host_trace = torch.empty((T, 13 + w, n), dtype=dtype).pin_memory()
    res = E.HostStepOut(b)
    E.rollout(a, ring, trace=dev_trace)
    E.rollout(b, ring.cpu().pin_memory(), trace=host_trace, out=res)
    same(a, b)
    assert torch.equal(host_trace, dev_trace.cpu())
    assert torch.equal(res.act, a.act.cpu()) and torch.equal(res.steps, a.steps.cpu())
