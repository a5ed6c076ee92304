"""ctypes binding of ``libuuvb200.so`` (the C ABI in ``include/uuv_b200.h``).

The library is built in-tree (``make`` / ``__graft_entry__.build()``) and
loaded from this package directory.  There is no fallback: if the library
is missing or a CUDA device is absent the product path raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UUV_B200_LIB") or os.path.join(_HERE, "libuuvb200.so")

MAX_ACT = 8
MAX_TYPES = 6
MLP_MAX_PARAMS = 128
MLP_MAX_WIDTH = 16
MLP_MAX_LAYERS = 4
MAX_DRAWS = 16
PW_MAX = 64

F32, F64 = 0, 1
PROPELLER, RUDDER, TILTROTOR = 0, 1, 2
ZERO_ORDER, FIRST_ORDER, DATA_DRIVEN = 0, 1, 2

# overlay keys (enum order of the header)
OV_KEYS = ("mass*", "volume*", "inertia*", "added_mass*", "damping*", "time_constant*",
           "thrust_coeff*", "cobm", "payload_mass*", "payload_position", "mount_position_jitter")
OV_INDEX = {k: i for i, k in enumerate(OV_KEYS)}
OV_COUNT = len(OV_KEYS)
OV_WIDTH = {k: 1 for k in OV_KEYS}
OV_WIDTH["payload_position"] = 3
OV_WIDTH["mount_position_jitter"] = 3 * MAX_ACT
OV_IDENTITY = {k: (1.0 if i <= OV_INDEX["thrust_coeff*"] else 0.0) for i, k in enumerate(OV_KEYS)}

ABI_VERSION = 7
MAX_RUNS = 8  # UUV_MAX_RUNS
DIST_UNIFORM, DIST_PIECEWISE, DIST_GAUSSIAN = 0, 1, 2
START_IDENTITY, START_BOX = 0, 1
CURRENT_NONE, CURRENT_RANDOM_HEADING, CURRENT_HEADING_DRAW = 0, 1, 2
TASK_STATION, TASK_TRACKING, TASK_DOCKING = 0, 1, 2
TRAJ_HELIX, TRAJ_LISSAJOUS = 0, 1
STATE_PAYLOAD_AT_ORIGIN = 1
RNG_PHILOX, RNG_PCG64 = 0, 1
RNG_MODES = {"philox": RNG_PHILOX, "pcg64": RNG_PCG64}
TR_NAMES = ("reward", "position_error", "attitude_error", "metric", "time", "contact_distance",
            "contact_speed", "contact_attitude")
# uuv_task_io.trace rows (UUV_TRACE_*): p(3) q(4) nu(6) reward t, then the command
TRACE_P, TRACE_Q, TRACE_NU, TRACE_REWARD, TRACE_T, TRACE_CMD = 0, 3, 7, 13, 14, 15
TF_NAMES = ("terminated", "truncated", "finished", "failure", "success", "diverged", "contact")
ST_NAMES = ("reward_sum", "finished", "success", "failure", "truncated", "metric_sum_finished",
            "diverged", "frames")


class Hull(C.Structure):
    _fields_ = [
        ("n_act", C.c_int32), ("flags", C.c_int32),
        ("kind", C.c_int32 * MAX_ACT), ("model", C.c_int32 * MAX_ACT),
        ("mlp_layers", C.c_int32), ("mlp_sizes", C.c_int32 * (MLP_MAX_LAYERS + 1)),
        ("mlp_relu", C.c_int32), ("pad_", C.c_int32),
        ("mass", C.c_double), ("volume", C.c_double), ("rho", C.c_double), ("g", C.c_double),
        ("r_g", C.c_double * 3), ("r_b", C.c_double * 3), ("inertia", C.c_double * 9),
        ("M_A", C.c_double * 36), ("D_lin", C.c_double * 36), ("D_quad", C.c_double * 36),
        ("limit", C.c_double * MAX_ACT), ("deadzone", C.c_double * MAX_ACT),
        ("reaction", C.c_double * MAX_ACT), ("thrust_coeff", C.c_double * MAX_ACT),
        ("time_constant", C.c_double * MAX_ACT),
        ("mount", (C.c_double * 3) * MAX_ACT), ("axis", (C.c_double * 3) * MAX_ACT),
        ("fin_xf", (C.c_double * 3) * MAX_ACT), ("fin_yf", (C.c_double * 3) * MAX_ACT),
        ("fin_area", C.c_double * MAX_ACT), ("fin_cla", C.c_double * MAX_ACT),
        ("fin_cd0", C.c_double * MAX_ACT), ("fin_kd", C.c_double * MAX_ACT),
        ("fin_stall", C.c_double * MAX_ACT), ("fin_rho", C.c_double * MAX_ACT),
        ("mlp", C.c_double * MLP_MAX_PARAMS),
    ]


class State(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("a_max", C.c_int32),
        ("n_envs", C.c_int64), ("ld", C.c_int64), ("env_offset", C.c_int64),
        ("p", C.c_void_p), ("q", C.c_void_p), ("nu", C.c_void_p), ("act", C.c_void_p),
        ("current_ned", C.c_void_p),
        ("steps", C.c_void_p), ("episodes", C.c_void_p), ("diverged", C.c_void_p),
        ("type_id", C.c_void_p), ("overlay", C.c_void_p), ("overlay_keys", C.c_void_p),
        ("n_slots", C.c_int32), ("slot", C.c_int32 * OV_COUNT), ("flags", C.c_int32),
        ("n_runs", C.c_int32), ("run_type", C.c_int32 * MAX_RUNS),
        ("run_start", C.c_int64 * MAX_RUNS),
    ]


class Draw(C.Structure):
    _fields_ = [("key", C.c_int32), ("dist", C.c_int32), ("n_draws", C.c_int32),
                ("pw_bins", C.c_int32), ("pw_offset", C.c_int32), ("pad_", C.c_int32),
                ("lo", C.c_double), ("hi", C.c_double), ("mu", C.c_double), ("sigma", C.c_double)]


class Sampler(C.Structure):
    _fields_ = [
        ("n_overlay", C.c_int32), ("current_mode", C.c_int32), ("start_mode", C.c_int32),
        ("rng_mode", C.c_int32),
        ("overlay", Draw * MAX_DRAWS), ("current_speed", Draw), ("current_heading", Draw),
        ("p_base", C.c_double * 3), ("p_lo", C.c_double * 3), ("p_hi", C.c_double * 3),
        ("eul_lo", C.c_double * 3), ("eul_hi", C.c_double * 3),
        ("nu_lo", C.c_double * 6), ("nu_hi", C.c_double * 6),
        ("pw_table", C.c_double * PW_MAX),
    ]


class Task(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("episode_length", C.c_int32), ("traj_kind", C.c_int32),
        ("obs_dim", C.c_int32),
        ("bounds", C.c_double), ("nu_max", C.c_double), ("fail_penalty", C.c_double),
        ("w_p", C.c_double), ("w_a", C.c_double), ("w_v", C.c_double), ("w_u", C.c_double),
        ("w_b", C.c_double), ("r_tol", C.c_double), ("speed_cap", C.c_double),
        ("dock_bonus", C.c_double), ("w_dock_dist", C.c_double), ("w_impact", C.c_double),
        ("w_level", C.c_double),
        ("target_p", C.c_double * 3), ("target_q", C.c_double * 4), ("success_tol", C.c_double),
        ("dock_centre", C.c_double * 3), ("dock_radius", C.c_double),
        ("traj_radius", C.c_double), ("traj_rate", C.c_double), ("traj_climb", C.c_double),
        ("traj_z0", C.c_double), ("traj_phase", C.c_double),
        ("traj_amp", C.c_double * 3), ("traj_rates", C.c_double * 3),
    ]


class TaskIO(C.Structure):
    _fields_ = [("prev_u", C.c_void_p), ("dev_sum", C.c_void_p), ("obs", C.c_void_p),
                ("obs_ld", C.c_int64), ("term_obs", C.c_void_p), ("real_out", C.c_void_p),
                ("flag_out", C.c_void_p), ("stats", C.c_void_p), ("trace", C.c_void_p),
                ("trace_ld", C.c_int64)]


class Policy(C.Structure):
    _fields_ = [("theta", C.c_void_p), ("theta_ld", C.c_int64), ("members", C.c_int32),
                ("slot", C.c_int32), ("ret", C.c_void_p), ("metric", C.c_void_p),
                ("success", C.c_void_p), ("pending", C.c_void_p), ("live", C.c_void_p),
                ("t", C.c_int32), ("pad_", C.c_int32)]


class HostOut(C.Structure):
    """uuv_host_out: pinned host result rows of one step (any field may be NULL)."""
    _fields_ = [("pose", C.c_void_p), ("act", C.c_void_p), ("steps", C.c_void_p),
                ("diverged", C.c_void_p)]


# DLPack (unversioned DLTensor, as declared in the header)
class DLDevice(C.Structure):
    _fields_ = [("device_type", C.c_int32), ("device_id", C.c_int32)]


class DLDataType(C.Structure):
    _fields_ = [("code", C.c_uint8), ("bits", C.c_uint8), ("lanes", C.c_uint16)]


class DLTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("device", DLDevice), ("ndim", C.c_int32),
                ("dtype", DLDataType), ("shape", C.POINTER(C.c_int64)),
                ("strides", C.POINTER(C.c_int64)), ("byte_offset", C.c_uint64)]


DL_P, DL_Q, DL_NU, DL_ACT, DL_CURRENT, DL_STEPS, DL_EPISODES, DL_DIVERGED, DL_COUNT = range(9)

_capsule_ptr = C.pythonapi.PyCapsule_GetPointer
_capsule_ptr.restype = C.c_void_p
_capsule_ptr.argtypes = [C.py_object, C.c_char_p]


class DLArg:
    """A torch tensor exported through DLPack (``torch.utils.dlpack.to_dlpack``),
    borrowed by one C call: ``.ptr`` is the capsule's ``DLManagedTensor*`` (its
    first member is the ``DLTensor``); the capsule, owned here, frees it when this
    object goes away.  Pass the DLArg ITSELF as the ctypes argument
    (``_as_parameter_``): the call's argument tuple then keeps the capsule alive --
    ``DLArg(t).ptr`` alone would let it be freed before the call runs."""

    __slots__ = ("capsule", "ptr", "_as_parameter_")

    def __init__(self, tensor):
        from torch.utils.dlpack import to_dlpack

        self.capsule = to_dlpack(tensor)
        self.ptr = _capsule_ptr(self.capsule, b"dltensor")
        self._as_parameter_ = C.c_void_p(self.ptr)


def dl(tensor):
    """DLArg of a tensor, or None for None."""
    return None if tensor is None else DLArg(tensor)


def dl_ptr(arg):
    return None if arg is None else arg.ptr


EXPORTS = {
    "uuv_last_error": (C.c_char_p, []),
    "uuv_abi_version": (C.c_int32, []),
    "uuv_abi_sizes": (None, [C.POINTER(C.c_int64)]),
    "uuv_ctx_create": (C.c_int, [C.POINTER(Hull), C.c_int32, C.POINTER(C.c_void_p)]),
    "uuv_ctx_set_hulls": (C.c_int, [C.c_void_p, C.POINTER(Hull), C.c_int32]),
    "uuv_ctx_destroy": (None, [C.c_void_p]),
    "uuv_step": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.c_int64, C.c_int32,
                           C.c_double, C.c_void_p]),
    "uuv_server_start": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_int32, C.c_double,
                                   C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "uuv_server_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(HostOut)]),
    "uuv_server_stop": (C.c_int, [C.c_void_p]),
    "uuv_server_stamps": (None, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "uuv_step_host": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.c_int64, C.c_void_p,
                                C.POINTER(HostOut), C.c_int32, C.c_double, C.c_void_p, C.c_int32]),
    "uuv_state_from_dlpack": (C.c_int, [C.POINTER(State), C.POINTER(C.c_void_p), C.c_int32]),
    "uuv_step_dl": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.c_int32, C.c_double,
                              C.c_void_p]),
    "uuv_rollout_dl": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_double, C.c_void_p, C.c_void_p,
                                 C.POINTER(HostOut), C.c_void_p]),
    "uuv_reset_dl": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.POINTER(Sampler),
                               C.c_uint64, C.c_void_p]),
    "uuv_task_step_dl": (C.c_int, [C.c_void_p, C.POINTER(State), C.POINTER(Task),
                                   C.POINTER(Sampler), C.c_uint64, C.c_void_p, C.c_int32,
                                   C.c_double, C.POINTER(TaskIO), C.c_void_p, C.c_void_p]),
    "uuv_reset": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.POINTER(Sampler),
                            C.c_uint64, C.c_void_p]),
    "uuv_task_step": (C.c_int, [C.c_void_p, C.POINTER(State), C.POINTER(Task), C.POINTER(Sampler),
                                C.c_uint64, C.c_void_p, C.c_int64, C.c_int32, C.c_double,
                                C.POINTER(TaskIO), C.c_void_p]),
    "uuv_policy_step": (C.c_int, [C.c_void_p, C.POINTER(State), C.POINTER(Task),
                                  C.POINTER(Sampler), C.c_uint64, C.POINTER(Policy), C.c_int32,
                                  C.c_double, C.POINTER(TaskIO), C.c_void_p]),
    "uuv_policy_episode": (C.c_int, [C.c_void_p, C.POINTER(State), C.POINTER(Task),
                                     C.POINTER(Sampler), C.c_uint64, C.POINTER(Policy), C.c_int32,
                                     C.c_int32, C.c_double, C.POINTER(TaskIO), C.c_void_p]),
    "uuv_task_reset": (C.c_int, [C.c_void_p, C.POINTER(State), C.POINTER(Task), C.POINTER(Sampler),
                                 C.c_uint64, C.c_void_p, C.c_double, C.POINTER(TaskIO),
                                 C.c_void_p]),
    "uuv_observe": (C.c_int, [C.c_void_p, C.POINTER(State), C.POINTER(Task), C.c_double,
                              C.POINTER(TaskIO), C.c_void_p]),
    "uuv_stats_blocks": (C.c_int64, [C.c_int64]),
    "uuv_rollout_stats": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p]),
    "uuv_derive_params": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]),
    "uuv_substep_terms": (C.c_int, [C.c_void_p, C.POINTER(State), C.c_void_p, C.c_int64,
                                    C.c_double, C.c_void_p, C.c_void_p]),
}

_lib = None


class NativeError(RuntimeError):
    pass


def load():
    """Load the in-tree library and check the ABI struct layout."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: build it with `make` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.uuv_abi_version() != ABI_VERSION:
        raise NativeError(f"ABI mismatch: library version {lib.uuv_abi_version()} != "
                          f"binding {ABI_VERSION}; rebuild with `make`")
    sizes = (C.c_int64 * 6)()
    lib.uuv_abi_sizes(sizes)
    want = [C.sizeof(Hull), C.sizeof(State), C.sizeof(Sampler), C.sizeof(Task), C.sizeof(TaskIO),
            C.sizeof(Policy)]
    if list(sizes) != want:
        raise NativeError(f"ABI mismatch: library struct sizes {list(sizes)} != binding {want}")
    _lib = lib
    return lib


def check(status: int, exc=NativeError):
    if status != 0:
        msg = load().uuv_last_error().decode(errors="replace")
        raise exc(msg)
