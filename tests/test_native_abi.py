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
    assert lib.uuv_abi_version() == N.ABI_VERSION == 4
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
