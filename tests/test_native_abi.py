"""CPU checks of the C ABI library and the host-side packing (no GPU calls)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2503_09203_b200 import _native as N
from paper_2503_09203_b200 import vehicles as pv
from paper_2503_09203_b200.engine import DeviceSampler, EngineError, pack_hull, spec_sampler
from paper_2503_09203_b200.randomization import DRParameter, Piecewise, Uniform, preset
from paper_2503_09203_b200.tasks import TaskConfig, start_box

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "uuv_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(uuv_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTS), set(names) ^ set(N.EXPORTS)


def test_abi_struct_sizes_and_version():
    lib = N.load()
    assert lib.uuv_abi_version() == N.ABI_VERSION == 7
    sizes = (C.c_int64 * 6)()
    lib.uuv_abi_sizes(sizes)
    assert list(sizes) == [C.sizeof(N.Hull), C.sizeof(N.State), C.sizeof(N.Sampler),
                           C.sizeof(N.Task), C.sizeof(N.TaskIO), C.sizeof(N.Policy)]


def test_ctx_create_validates_hulls():
    lib = N.load()
    h = pack_hull(pv.load_vehicle("bluerov"))
    ctx = C.c_void_p()
    assert lib.uuv_ctx_create(C.byref(h), 1, C.byref(ctx)) == 0
    lib.uuv_ctx_destroy(ctx)
    bad = pack_hull(pv.load_vehicle("bluerov"))
    bad.mass = -1.0
    assert lib.uuv_ctx_create(C.byref(bad), 1, C.byref(ctx)) == 1
    assert b"mass" in lib.uuv_last_error()
    assert lib.uuv_ctx_create(C.byref(h), 0, C.byref(ctx)) == 4


def test_step_rejects_bad_arguments_without_gpu():
    lib = N.load()
    h = pack_hull(pv.load_vehicle("bluerov"))
    ctx = C.c_void_p()
    assert lib.uuv_ctx_create(C.byref(h), 1, C.byref(ctx)) == 0
    st = N.State()
    st.dtype, st.a_max, st.n_envs, st.ld = 0, 6, 4, 2  # ld < n
    assert lib.uuv_step(ctx, C.byref(st), None, 6, 1, 0.02, None) == 2
    assert b"ld" in lib.uuv_last_error()
    lib.uuv_ctx_destroy(ctx)


@pytest.mark.parametrize("name", pv.BUILTIN_VEHICLES)
def test_pack_hull_layout(name):
    veh = pv.load_vehicle(name)
    h = pack_hull(veh)
    assert h.n_act == veh.action_dim
    for j, a in enumerate(veh.actuators):
        assert h.kind[j] == pv.KIND_CODE[a.kind]
        assert h.limit[j] == a.state_limit
        if a.kind == "tiltrotor":
            ax = pv.tilt_rotation(a.mount_axis, a.tilt_axis, a.tilt_angle_default)
            assert np.allclose(list(h.axis[j]), ax, atol=0)
    assert list(h.M_A)[0] == veh.coeffs.M_A[0, 0]


def test_pack_hull_rotor_net():
    import variants

    veh = variants.build("rotor_mix", pv, pv, pv, pv.load_vehicle("bluerov"))
    h = pack_hull(veh)
    assert h.mlp_layers == 2 and list(h.mlp_sizes)[:3] == [2, 8, 1]
    assert h.model[0] == 2 and h.model[2] == 0 and h.reaction[4] == 3.0e-6
    assert h.mlp[0] == 1.5 and h.mlp[16 + 8] == 0.8


def test_sampler_packing_follows_sorted_keys():
    spec = preset("train")
    smp = spec_sampler(spec, start_box(TaskConfig(task="docking"))).pack()
    keys = [N.OV_KEYS[smp.overlay[d].key] for d in range(smp.n_overlay)]
    assert keys == ["added_mass*", "cobm", "damping*", "inertia*", "mass*", "payload_mass*",
                    "volume*"]
    assert smp.current_mode == N.CURRENT_RANDOM_HEADING
    assert smp.current_speed.hi == 0.5 and smp.start_mode == N.START_BOX
    assert list(smp.p_lo) == [-1.5, -1.5, -2.5]


def test_sampler_piecewise_table():
    spec = {"mass*": DRParameter("mass*", Piecewise([0.5, 1.0, 1.5], [1.0, 3.0]))}
    smp = DeviceSampler(spec).pack()
    d = smp.overlay[0]
    assert d.dist == N.DIST_PIECEWISE and d.pw_bins == 2
    tbl = list(smp.pw_table)[:5]
    assert tbl[:3] == [0.5, 1.0, 1.5] and tbl[3] == 0.25 and tbl[4] == 1.0


def test_hull_rejects_too_many_actuators():
    veh = pv.load_vehicle("bluerov_heavy")
    import copy

    big = copy.deepcopy(veh)
    big.actuators = big.actuators + [copy.deepcopy(big.actuators[0])]
    with pytest.raises(EngineError):
        pack_hull(big)


def _dl_fields(n=5, a=6, ld=32, dtype=None, device="cpu"):
    import torch

    dtype = dtype or torch.float32
    soa = torch.zeros((13 + a, ld), dtype=dtype, device=device)
    f = [soa[0:3, :n].t(), soa[3:7, :n].t(), soa[7:13, :n].t(), soa[13:, :n].t(), None,
         torch.zeros(ld, dtype=torch.int32, device=device)[:n],
         torch.zeros(ld, dtype=torch.int32, device=device)[:n],
         torch.zeros(ld, dtype=torch.bool, device=device)[:n]]
    return f


def _bind(fields, count=None):
    lib = N.load()
    args = [N.dl(t) for t in fields]
    ptrs = (C.c_void_p * len(args))(*[N.dl_ptr(x) for x in args])
    st = N.State()
    return lib.uuv_state_from_dlpack(C.byref(st), ptrs, count or len(args)), st


def test_dlpack_state_validation_without_gpu():
    """uuv_state_from_dlpack validates the DLPack fields in C (device checked before any
    CUDA call, so CPU tensors are refused here without a GPU)."""
    import torch

    lib = N.load()
    status, _ = _bind(_dl_fields(), count=3)
    assert status == N_ERR_ARG and b"DLPack fields" in lib.uuv_last_error()
    f = _dl_fields()
    f[N.DL_STEPS] = None
    status, _ = _bind(f)
    assert status == N_ERR_ARG and b"steps: null" in lib.uuv_last_error()
    status, _ = _bind(_dl_fields())  # CPU tensors
    assert status == N_ERR_ARG and b"not CUDA" in lib.uuv_last_error()
    f = _dl_fields(a=9, ld=32)
    status, _ = _bind(f)
    assert status == N_ERR_SHAPE and b"act" in lib.uuv_last_error()
    f = _dl_fields(dtype=torch.float16)
    status, _ = _bind(f)
    assert status == N_ERR_ARG and b"float32 or float64" in lib.uuv_last_error()


N_ERR_ARG, N_ERR_SHAPE = 1, 2


def test_dlarg_exports_the_tensor_layout():
    """DLArg hands the C side torch's own DLPack export (shape, strides, dtype codes)."""
    import torch

    soa = torch.zeros((3, 64))
    arg = N.DLArg(soa[:, :40].t())
    t = C.cast(arg.ptr, C.POINTER(N.DLTensor)).contents
    assert t.ndim == 2 and (t.shape[0], t.shape[1]) == (40, 3)
    assert (t.strides[0], t.strides[1]) == (1, 64)
    assert (t.dtype.code, t.dtype.bits, t.dtype.lanes) == (2, 32, 1)
    assert t.device.device_type == 1  # kDLCPU
    barg = N.DLArg(torch.zeros(4, dtype=torch.bool))  # keep the capsule alive while reading
    b = C.cast(barg.ptr, C.POINTER(N.DLTensor)).contents
    assert (b.dtype.code, b.dtype.bits) == (6, 8)


def test_dlarg_is_passed_as_the_ctypes_argument():
    """A temporary DLArg passed directly stays alive for the call (``_as_parameter_``): the C
    side reads its DLTensor (here: refuses its CPU device) -- no GPU call is reached."""
    import torch

    lib = N.load()
    h = pack_hull(pv.load_vehicle("bluerov"))
    ctx = C.c_void_p()
    assert lib.uuv_ctx_create(C.byref(h), 1, C.byref(ctx)) == 0
    st = N.State()
    st.dtype, st.a_max, st.n_envs, st.ld = 0, 6, 4, 32
    for name in ("p", "q", "nu", "act", "steps", "episodes", "diverged"):
        setattr(st, name, 256)  # never dereferenced: validation fails first
    for k in range(N.OV_COUNT):
        st.slot[k] = -1
    status = lib.uuv_step_dl(ctx, C.byref(st), N.DLArg(torch.zeros((4, 6))), 1, 0.02, None)
    assert status == N_ERR_ARG and b"commands: DLPack device type 1" in lib.uuv_last_error()
    status = lib.uuv_step_dl(ctx, C.byref(st), N.DLArg(torch.zeros((5, 6))), 1, 0.02, None)
    assert b"not CUDA" in lib.uuv_last_error()
    lib.uuv_ctx_destroy(ctx)
