"""The drop-in boundary on the GPU: host result rows, DLPack tensors, the reference binding.

* ``uuv_step_host`` / the step server return the whole step result (p, q, nu,
  act, steps, diverged — what the reference's in-place step_batch mutates,
  engine.py:418, 444-449) from EVERY step-kernel build: single vehicle with and
  without DR, the mixed-fleet kernel, the 96-register large-batch build, and the
  copy-engine path.
* The C ABI taking DLPack tensors (``uuv_state_from_dlpack``, ``uuv_step_dl``,
  ``uuv_reset_dl``, ``uuv_task_step_dl``) with torch capsules passed through
  ctypes, including its dtype / device / shape / stride validation.
* The INTEGRATION.md §2 binding (``refbind``) executed against the unmodified
  reference's own BatchState (baseline/_ref), compared with the reference's
  own step_batch.
"""

import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
from conftest import product_vehicle

from paper_2503_09203_b200 import _native as N
from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.randomization import DRParameter, Uniform

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dr_spec(keys=("mass*", "damping*", "thrust_coeff*", "volume*")):
    return {k: DRParameter(k, Uniform(0.8, 1.2)) for k in keys}


def make_pair(case, dtype):
    """Two identical batches for a kernel path of uuv_step (see dispatch_step)."""
    if case == "fleet":
        vehs = [product_vehicle(v) for v in ("bluerov", "lauv", "hauv")]
        n = 3000
        counts = [1000, 1000, 1000]

        def make():
            st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n), master_seed=2,
                                    dtype=dtype)
            E.reset_envs(st, np.ones(n, bool), E.spec_sampler(dr_spec(("mass*",))))
            return st
    else:
        n = {"nodr": 1000, "dr": 4096, "hi": 131_072}[case]
        spec = None if case == "nodr" else dr_spec()

        def make():
            st = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=n),
                              master_seed=2, dtype=dtype)
            E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
            return st
    return make(), make(), n


def expect_out(res, st):
    w = E._cmd_width(st)
    assert torch.equal(res.p, st.p.cpu()) and torch.equal(res.q, st.q.cpu())
    assert torch.equal(res.nu, st.nu.cpu())
    assert torch.equal(res.act, st.act[:, :w].cpu())
    assert torch.equal(res.steps, st.steps.cpu())
    assert torch.equal(res.diverged, st.diverged.cpu())


@pytest.mark.parametrize("case,dtype", [("nodr", torch.float32), ("nodr", torch.float64),
                                        ("dr", torch.float32), ("dr", torch.float64),
                                        ("fleet", torch.float32), ("fleet", torch.float64),
                                        ("hi", torch.float32)])
def test_host_out_from_every_step_build(case, dtype):
    """step_batch(pinned host commands, out=HostStepOut) == the device step, every field,
    bit for bit -- frozen (diverged) rows included."""
    a, b, n = make_pair(case, dtype)
    w = E._cmd_width(a)
    res = E.HostStepOut(b)
    pose = torch.empty((13, n), dtype=dtype).pin_memory()
    g = torch.Generator().manual_seed(0)
    for t in range(4):
        hc = (torch.rand((n, w), generator=g, dtype=torch.float64) * 2.2 - 1.1).to(dtype)
        if t == 1:
            hc[5, 0] = float("nan")  # env 5 diverges, then stays frozen
        hc = hc.pin_memory()
        E.step_batch(a, hc.cuda())
        E.step_batch(b, hc, out=res)
        for k in ("p", "q", "nu", "act", "steps", "diverged"):
            assert torch.equal(getattr(a, k), getattr(b, k)), (case, t, k)
        expect_out(res, a)
        E.step_batch(a, hc.cuda())
        E.step_batch(b, hc, pose_out=pose)  # the pose-only shorthand
        assert torch.equal(pose, torch.cat([a.p, a.q, a.nu], dim=1).T.cpu())
    assert bool(res.diverged[5]) and int(res.steps[5]) == 7  # the last out= step is the 7th
    assert res.nbytes == n * (13 * res.pose.element_size() + w * res.pose.element_size() + 5)


def test_host_out_copy_engine_path():
    """UUV_HOST_STEP=copy: the same results through cudaMemcpy2DAsync of every field."""
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests/golden')
from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.vehicles import load_vehicle
n = 777
a, b = (E.make_batch(load_vehicle('hauv'), E.SimConfig(batch_size=n), master_seed=1)
        for _ in range(2))
for st in (a, b):
    E.reset_envs(st, np.ones(n, bool))
res = E.HostStepOut(b)
hc = (torch.rand((n, 8), generator=torch.Generator().manual_seed(3)) * 2 - 1).pin_memory()
for t in range(3):
    E.step_batch(a, hc.cuda()); E.step_batch(b, hc, out=res)
    assert torch.equal(res.p, a.p.cpu()) and torch.equal(res.nu, a.nu.cpu())
    assert torch.equal(res.act, a.act.cpu()) and torch.equal(res.steps, a.steps.cpu())
    assert torch.equal(res.diverged, a.diverged.cpu())
print('copy-path ok')
"""
    env = dict(os.environ, UUV_HOST_STEP="copy")
    r = subprocess.run([sys.executable, "-c", code, ROOT], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "copy-path ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_step_server_returns_the_whole_result(dtype):
    """serve(): HostStepOut rows (act, steps, diverged too) == launched steps, mixed fleet."""
    a, b, n = make_pair("fleet", dtype)
    w = E._cmd_width(a)
    res = E.HostStepOut(b)
    g = torch.Generator().manual_seed(4)
    cmds = [(torch.rand((n, w), generator=g, dtype=torch.float64) * 2 - 1).to(dtype).pin_memory()
            for _ in range(5)]
    cmds[2][11, 1] = float("nan")
    assert torch.equal(res.p, res.p)  # torch host kernels loaded before the server starts
    with E.serve(b):
        for t in range(5):
            E.step_batch(a, cmds[t].cuda())
            E.step_batch(b, cmds[t], out=res)
            expect_out(res, a)
        partial = E.HostStepOut(b, fields=("steps", "diverged"))
        E.step_batch(a, cmds[0].cuda())
        E.step_batch(b, cmds[0], out=partial)
        assert torch.equal(partial.steps, a.steps.cpu()) and partial.pose is None
    assert bool(a.diverged[11])


# ------------------------------------------------------------------ DLPack through ctypes


def soa_fields(n, a, dtype, ld=None, dev="cuda"):
    ld = ld or max(32, -(-n // 32) * 32)
    soa = torch.zeros((13 + a, ld), dtype=dtype, device=dev)
    soa[3] = 1.0
    return soa, [soa[0:3, :n].t(), soa[3:7, :n].t(), soa[7:13, :n].t(), soa[13:, :n].t(), None,
                 torch.zeros(ld, dtype=torch.int32, device=dev)[:n],
                 torch.full((ld,), -1, dtype=torch.int32, device=dev)[:n],
                 torch.zeros(ld, dtype=torch.bool, device=dev)[:n]]


def bind(fields):
    lib = N.load()
    args = [N.dl(t) for t in fields]
    ptrs = (C.c_void_p * len(args))(*[N.dl_ptr(x) for x in args])
    st = N.State()
    for k in range(N.OV_COUNT):
        st.slot[k] = -1
    st.flags = N.STATE_PAYLOAD_AT_ORIGIN
    status = lib.uuv_state_from_dlpack(C.byref(st), ptrs, len(args))
    return status, st


def last_error():
    return N.load().uuv_last_error().decode()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_dlpack_capsules_through_ctypes(dtype):
    """A caller holding only torch tensors: capsules -> C ABI -> kernel, == step_batch."""
    lib = N.load()
    veh = product_vehicle("bluerov_heavy")
    n, a = 1000, veh.action_dim
    soa, fields = soa_fields(n, a, dtype)
    status, cst = bind(fields)
    assert status == 0, last_error()
    assert (cst.n_envs, cst.ld, cst.a_max) == (n, soa.shape[1], a)
    hull = E.pack_hull(veh)
    ctx = C.c_void_p()
    assert lib.uuv_ctx_create(C.byref(hull), 1, C.byref(ctx)) == 0
    stream = torch.cuda.current_stream().cuda_stream
    smp = E.DeviceSampler().pack()
    assert lib.uuv_reset_dl(ctx, C.byref(cst), None, C.byref(smp), 0, stream) == 0
    ref = E.make_batch(veh, E.SimConfig(batch_size=n), dtype=dtype)
    E.reset_envs(ref, np.ones(n, bool))
    g = torch.Generator(device="cuda").manual_seed(0)
    for t in range(5):
        cmd = (torch.rand((n, a), device="cuda", generator=g) * 2 - 1).to(dtype)
        arg = N.DLArg(cmd)
        assert lib.uuv_step_dl(ctx, C.byref(cst), arg, 1, 0.02, stream) == 0, last_error()
        E.step_batch(ref, cmd)
    torch.cuda.synchronize()
    assert torch.equal(fields[0], ref.p) and torch.equal(fields[2], ref.nu)
    assert torch.equal(fields[5], ref.steps) and torch.equal(fields[6], ref.episodes)

    def err(cmd):
        return lib.uuv_step_dl(ctx, C.byref(cst), N.DLArg(cmd), 1, 0.02, stream)

    other = torch.float64 if dtype == torch.float32 else torch.float32
    assert err(torch.zeros((n, a), dtype=other, device="cuda")) == 1
    assert "dtype" in last_error()
    assert err(torch.zeros((n, a + 1), dtype=dtype, device="cuda")) == 2
    assert "expected shape" in last_error()
    assert err(torch.zeros((a, n), dtype=dtype, device="cuda").t()) == 2
    assert "column stride" in last_error()
    assert err(torch.zeros((n, a), dtype=dtype)) == 1 and "not CUDA" in last_error()
    wide = torch.zeros((n, 16), dtype=dtype, device="cuda")[:, :a]  # row stride 16: accepted
    assert err(wide) == 0
    bad_mask = torch.ones(n, dtype=torch.float32, device="cuda")
    assert lib.uuv_reset_dl(ctx, C.byref(cst), N.DLArg(bad_mask), C.byref(smp), 0,
                            stream) == 1
    assert "bool or uint8" in last_error()
    lib.uuv_ctx_destroy(ctx)


def test_dlpack_state_layout_is_validated():
    """SoA strides, shared component stride, per-field dtype and device checked in C."""
    n, a = 100, 6
    _, f = soa_fields(n, a, torch.float32)
    f2 = list(f)
    f2[0] = torch.zeros((n, 3), device="cuda")  # row-major (N, 3): env stride 3
    assert bind(f2)[0] == 2 and "env stride" in last_error()
    f2 = list(f)
    f2[1] = torch.zeros((4, 256), device="cuda")[:, :n].t()  # different component stride
    assert bind(f2)[0] == 2 and "component stride" in last_error()
    f2 = list(f)
    f2[2] = f2[2].double()
    assert bind(f2)[0] == 1 and "dtype differs" in last_error()
    f2 = list(f)
    f2[5] = torch.zeros(n, dtype=torch.int64, device="cuda")
    assert bind(f2)[0] == 1 and "int32" in last_error()
    f2 = list(f)
    f2[7] = torch.zeros(n + 1, dtype=torch.bool, device="cuda")
    assert bind(f2)[0] == 2 and "diverged" in last_error()
    f2 = list(f)
    f2[4] = torch.zeros((3, 256), device="cuda")[:, :n].t()  # current_ned, other ld
    assert bind(f2)[0] == 2 and "current_ned" in last_error()


def test_task_step_dl_writes_the_observation_tensor():
    from paper_2503_09203_b200.tasks import TaskConfig, make_env

    task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr")
    n = 512
    envs = [make_env(task, E.SimConfig(batch_size=n), seed=3) for _ in range(2)]
    for e in envs:
        e.reset()
    g = torch.Generator(device="cuda").manual_seed(1)
    for _ in range(30):
        u = torch.rand((n, 8), device="cuda", generator=g) * 2 - 1
        o0, r0, te0, tr0, _ = envs[0].step(u)
        o1, r1, te1, tr1, _ = envs[1].step(u)
        assert torch.equal(o0, o1) and torch.equal(r0, r1) and torch.equal(te0, te1)
    # obs tensor of the wrong width is refused by the C side
    st = envs[0].state
    lib = N.load()
    bad = torch.empty((n, envs[0].obs_dim + 1), device="cuda")
    io = envs[0]._io(None)
    status = lib.uuv_task_step_dl(st._ctx, C.byref(st._cstate()), C.byref(envs[0]._task_c),
                                  C.byref(envs[0]._sampler_c), 3, N.DLArg(u), 1, 0.02,
                                  C.byref(io), N.DLArg(bad), st._stream())
    assert status == 2 and "obs" in last_error()


# ------------------------------------------------------------------ the reference, bound


def reference_engine():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "uuvsim")):
        pytest.skip("the unmodified reference is not installed in baseline/_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import uuvsim.engine as RE
    import uuvsim.randomization as RD
    import uuvsim.vehicles as RV
    from uuvsim.kinematics import Pose

    return RE, RD, RV, Pose


def test_integration_stub_against_the_unmodified_reference():
    """the reference's own BatchState (PCG64 streams, its own DR draws and
    overlay math) stepped through refbind == the reference's own step_batch, float64."""
    from paper_2503_09203_b200 import refbind

    RE, RD, RV, Pose = reference_engine()
    veh = RV.load_vehicle("bluerov")
    n = 256
    spec = RD.make_spec([RD.DRParameter(k, RD.Uniform(0.8, 1.2))
                         for k in ("damping*", "mass*", "thrust_coeff*", "volume*")])

    def sampler(i, ep, rng):
        return RE.EnvInit(pose=Pose(p=rng.uniform(-1, 1, 3)), nu=rng.uniform(-0.2, 0.2, 6),
                          overlay=RD.sample_overlay(spec, rng),
                          current_ned=rng.uniform(-0.2, 0.2, 3) if i % 2 else np.zeros(3))

    states = []
    for _ in range(2):
        st = RE.make_batch(veh, RE.SimConfig(batch_size=n, substeps=2), master_seed=11)
        RE.reset_envs(st, np.ones(n, bool), sampler)
        states.append(st)
    plain, bound = states
    original = refbind.install(RE)
    try:
        refbind.bind(bound)
        cmds = np.random.default_rng(0).uniform(-1.0, 1.0, (30, n, veh.action_dim))
        for t in range(30):
            if t == 15:  # a partial reset mid-run: new episodes, new overlays
                mask = np.random.default_rng(t).random(n) < 0.3
                for st in states:
                    RE.reset_envs(st, mask, sampler)
            RE.step_batch(plain, cmds[t])  # unbound: the reference itself
            RE.step_batch(bound, cmds[t])
            for k in ("p", "q", "nu", "act"):
                a, b = getattr(plain, k), getattr(bound, k)
                err = np.abs(a - b).max(axis=1) / np.maximum(np.abs(a).max(axis=1), 1e-300)
                assert err.max() <= 1e-10, (t, k, err.max())
            assert np.array_equal(plain.steps, bound.steps)
            assert np.array_equal(plain.diverged, bound.diverged)
        with pytest.raises(RE.EngineError, match="commands"):
            RE.step_batch(bound, np.zeros((n, 5)))
    finally:
        RE.step_batch = original
