"""Batched lockstep engine over the B200 kernels — the reference API, on device.

Drop-in for ``uuvsim/engine.py``: ``SimConfig`` (63-77), ``make_batch``
(298-320), ``step_batch`` (465-484), ``reset_envs`` (487-512),
``env_snapshot`` (515-527), ``throughput_probe`` (541-564), ``EnvInit`` /
``default_sampler`` (252-266), ``BatchState.env_rng`` (291-295).

State fields keep the reference names and shapes — ``p`` (N,3), ``q``
(N,4) wxyz body->NED, ``nu`` (N,6), ``act`` (N,A), ``current_ned`` (N,3),
``steps`` / ``episodes`` (N,), ``diverged`` (N,) — but are torch CUDA tensors
that view a struct-of-arrays HBM layout (component-major, rows padded to a
multiple of 32), so every kernel load is a fully coalesced 128-byte line.
``steps`` / ``episodes`` are int32.  float32 is the default compute dtype;
``dtype=torch.float64`` selects the validation build (parity ~1e-12).

Every step is ONE kernel launch (``uuv_step_dl``: the commands cross the C ABI
as a DLPack tensor, the state fields were bound once through
``uuv_state_from_dlpack``) with K substeps fused in registers; no host
synchronisation happens inside ``step_batch``.

Randomness (behaviour change vs the reference, opt-in to match it): per-(seed,
env, episode) streams default to the north star's counter-based Philox4x64-10,
``Philox(key=[seed, env_offset + i], counter=[0, episode, 0, 0])``; the
unmodified reference draws from ``PCG64(SeedSequence(seed, spawn_key=(env,
episode)))`` (engine.py:291-295).  Pass ``rng="pcg64"`` to ``make_batch`` /
``make_env`` to reproduce the reference's episodes and DR draws bit for bit
(both streams are restated on the device).
"""

from __future__ import annotations

import ctypes as C
import math
import time
import weakref
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _native as N
from .randomization import CURRENT_KEYS, encodable
from .vehicles import (
    DATA_DRIVEN, FIRST_ORDER, KIND_CODE, MODEL_CODE, RUDDER, TILTROTOR, VehicleConfig,
    fin_basis, tilt_rotation, validate_overlay,
)

M64 = (1 << 64) - 1
_ALIGN = 32

try:  # the raw cudaStream_t of the current stream without building a Stream object
    _get_raw_stream = torch._C._cuda_getCurrentRawStream

    def _raw_stream(index):
        return _get_raw_stream(index)
except AttributeError:  # pragma: no cover
    def _raw_stream(index):
        return torch.cuda.current_stream(index).cuda_stream


class EngineError(ValueError):
    pass


@dataclass
class SimConfig:
    dt: float = 0.02
    substeps: int = 1
    batch_size: int = 1
    workers: int = 1  # accepted for API parity; results never depend on it

    def __post_init__(self):
        if self.dt <= 0:
            raise EngineError(f"dt must be > 0, got {self.dt}")
        if self.substeps < 1:
            raise EngineError(f"substeps must be >= 1, got {self.substeps}")
        if self.batch_size < 1:
            raise EngineError(f"batch_size must be >= 1, got {self.batch_size}")
        if self.workers < 1:
            raise EngineError(f"workers must be >= 1, got {self.workers}")


@dataclass
class Pose:
    p: np.ndarray = field(default_factory=lambda: np.zeros(3))
    q: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0, 0.0]))

    def __post_init__(self):
        self.p = np.asarray(self.p, dtype=float)
        self.q = np.asarray(self.q, dtype=float)


@dataclass
class EnvInit:
    pose: Pose
    nu: np.ndarray = field(default_factory=lambda: np.zeros(6))
    overlay: dict = field(default_factory=dict)
    current_ned: np.ndarray = field(default_factory=lambda: np.zeros(3))


InitSampler = Callable[[int, int, np.random.Generator], EnvInit]


def default_sampler(env_index: int, episode: int, rng) -> EnvInit:
    """Identity pose, zero velocity, no overlay, no current (engine.py:265-266)."""
    return EnvInit(pose=Pose())


def philox_generator(seed: int, env_index: int, episode: int) -> np.random.Generator:
    """Host twin of the device Philox stream (same bits as the reset kernel)."""
    return np.random.Generator(np.random.Philox(
        key=np.array([int(seed) & M64, int(env_index) & M64], dtype=np.uint64),
        counter=np.array([0, int(episode) & M64, 0, 0], dtype=np.uint64)))


def pcg64_generator(seed: int, env_index: int, episode: int) -> np.random.Generator:
    """The reference's own stream, PCG64(SeedSequence(seed, spawn_key=(env, episode)))
    (engine.py:291-295); the reset kernel restates it bit for bit (rng="pcg64")."""
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence(int(seed) & M64, spawn_key=(int(env_index), int(episode)))))


RNG_GENERATORS = {"philox": philox_generator, "pcg64": pcg64_generator}


# ================================================================ hull packing


def pack_hull(veh: VehicleConfig) -> N.Hull:
    """Compile one vehicle into the ABI hull table (compile_layout, engine.py:129-189)."""
    acts = veh.actuators
    A = len(acts)
    if not 1 <= A <= N.MAX_ACT:
        raise EngineError(f"{veh.name}: {A} actuators, the device build supports 1..{N.MAX_ACT}")
    h = N.Hull()
    h.n_act = A
    rb, co = veh.rb, veh.coeffs
    h.mass, h.volume, h.rho, h.g = rb.mass, rb.displaced_volume, co.fluid_density, co.gravity
    for k in range(3):
        h.r_g[k], h.r_b[k] = rb.r_g[k], rb.r_b[k]
    for k, v in enumerate(np.asarray(rb.inertia, float).ravel()):
        h.inertia[k] = v
    for name in ("M_A", "D_lin", "D_quad"):
        dst = getattr(h, name)
        for k, v in enumerate(np.asarray(getattr(co, name), float).ravel()):
            dst[k] = v
    nets = []
    for j, a in enumerate(acts):
        h.kind[j] = KIND_CODE[a.kind]
        h.model[j] = MODEL_CODE[a.rotor_model]
        h.limit[j] = a.state_limit
        h.deadzone[j] = a.deadzone
        h.reaction[j] = a.reaction_coeff
        h.thrust_coeff[j] = a.thrust_coeff
        h.time_constant[j] = a.time_constant
        axis = tilt_rotation(a.mount_axis, a.tilt_axis, a.tilt_angle_default) \
            if a.kind == TILTROTOR else a.mount_axis
        for c in range(3):
            h.mount[j][c] = a.mount_position[c]
            h.axis[j][c] = axis[c]
        if a.kind == RUDDER:
            xf, yf = fin_basis(a.mount_axis)
            for c in range(3):
                h.fin_xf[j][c], h.fin_yf[j][c] = xf[c], yf[c]
            g = a.rudder
            h.fin_area[j], h.fin_cla[j], h.fin_cd0[j] = g.area, g.c_l_alpha, g.c_d0
            h.fin_kd[j], h.fin_stall[j], h.fin_rho[j] = g.k_d, g.stall_angle, g.fluid_density
        if a.rotor_model == DATA_DRIVEN:
            if a.mlp is None:
                raise EngineError(f"actuator {j}: data_driven model has no weights")
            if all(a.mlp is not n for n in nets):
                nets.append(a.mlp)
    if len(nets) > 1:
        raise EngineError(f"{veh.name}: the device build supports one rotor network per vehicle")
    if nets:
        net = nets[0]
        sizes = list(net.layer_sizes)
        if len(sizes) - 1 > N.MLP_MAX_LAYERS or max(sizes) > N.MLP_MAX_WIDTH:
            raise EngineError(f"{veh.name}: rotor network {sizes} exceeds the device envelope")
        flat = np.concatenate([np.concatenate([np.asarray(w, float).ravel(),
                                               np.asarray(b, float).ravel()])
                               for w, b in zip(net.weights, net.biases)])
        if flat.size > N.MLP_MAX_PARAMS:
            raise EngineError(f"{veh.name}: rotor network has {flat.size} > "
                              f"{N.MLP_MAX_PARAMS} parameters")
        h.mlp_layers = len(sizes) - 1
        for k, s in enumerate(sizes):
            h.mlp_sizes[k] = s
        h.mlp_relu = 1 if net.activation == "relu" else 0
        for k, v in enumerate(flat):
            h.mlp[k] = v
    return h


# ================================================================ declarative samplers


@dataclass
class DeviceSampler:
    """An episode sampler the reset kernel evaluates (tasks/core.py:282-289).

    ``overlay_spec``: DR spec without current keys, drawn in sorted key order;
    ``current_spec``: spec holding ``current_velocity`` [+ ``current_direction``];
    ``start``: None (identity pose) or the 7-tuple of ``tasks.start_box``.
    """

    overlay_spec: dict | None = None
    current_spec: dict | None = None
    start: tuple | None = None

    def keys(self):
        return sorted(self.overlay_spec) if self.overlay_spec else []

    def pack(self) -> N.Sampler:
        s = N.Sampler()
        pw = []

        def fill(d: N.Draw, key_code, dist, n_draws):
            d.key = key_code
            d.n_draws = n_draws
            if not encodable(dist):
                raise EngineError(f"{type(dist).__name__}: not a device-encodable distribution "
                                  "(use a sampler callable for the host reset path)")
            dist.encode(d, pw)

        keys = self.keys()
        if len(keys) > N.MAX_DRAWS:
            raise EngineError(f"at most {N.MAX_DRAWS} overlay keys")
        s.n_overlay = len(keys)
        for d, key in enumerate(keys):
            p = self.overlay_spec[key]
            fill(s.overlay[d], N.OV_INDEX[key], p.distribution, 3 if p.vector_valued else 1)
        cs = self.current_spec or {}
        if "current_velocity" in cs:
            fill(s.current_speed, 0, cs["current_velocity"].distribution, 1)
            if "current_direction" in cs:
                s.current_mode = N.CURRENT_HEADING_DRAW
                fill(s.current_heading, 0, cs["current_direction"].distribution, 1)
            else:
                s.current_mode = N.CURRENT_RANDOM_HEADING
        if self.start is not None:
            s.start_mode = N.START_BOX
            base, plo, phi, elo, ehi, nlo, nhi = self.start
            for c in range(3):
                s.p_base[c], s.p_lo[c], s.p_hi[c] = base[c], plo[c], phi[c]
                s.eul_lo[c], s.eul_hi[c] = elo[c], ehi[c]
            for c in range(6):
                s.nu_lo[c], s.nu_hi[c] = nlo[c], nhi[c]
        if len(pw) > N.PW_MAX:
            raise EngineError(f"piecewise tables exceed {N.PW_MAX} entries")
        for k, v in enumerate(pw):
            s.pw_table[k] = v
        return s


def spec_sampler(dr_spec: dict | None, start=None) -> DeviceSampler:
    """Device sampler for a DR spec (current keys split off) and a start box."""
    if dr_spec is None:
        return DeviceSampler(None, None, start)
    dyn = {k: p for k, p in dr_spec.items() if k not in CURRENT_KEYS}
    cur = {k: p for k, p in dr_spec.items() if k in CURRENT_KEYS}
    return DeviceSampler(dyn or None, cur or None, start)


_IDENTITY = DeviceSampler()


# ================================================================ batch state


class ParamsView:
    """Per-env parameters (BatchParams, engine.py:193-234), derived on device from
    the hull table and the overlay record; float64, read-only copies."""

    def __init__(self, state: "BatchState"):
        self._st = state

    def _derive(self):
        st = self._st
        n, am = st.n_envs, st.a_max
        dev = st.device
        out12 = torch.empty((n, 12), dtype=torch.float64, device=dev)
        minv = torch.empty((n, 6, 6), dtype=torch.float64, device=dev)
        ct_tau = torch.empty((n, 2, am), dtype=torch.float64, device=dev)
        mounts = torch.empty((n, am, 3), dtype=torch.float64, device=dev)
        lib = N.load()
        N.check(lib.uuv_derive_params(st._ctx, C.byref(st._cstate()), out12.data_ptr(),
                                      minv.data_ptr(), ct_tau.data_ptr(), mounts.data_ptr(),
                                      st._stream()), EngineError)
        return out12, minv, ct_tau, mounts

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        o12, minv, ct_tau, mounts = self._derive()
        table = {"mass": o12[:, 0], "volume": o12[:, 1], "r_g": o12[:, 2:5], "r_b": o12[:, 5:8],
                 "weight": o12[:, 8], "buoyancy": o12[:, 9], "added_mass_scale": o12[:, 10],
                 "damping_scale": o12[:, 11], "M_inv": minv, "thrust_coeff": ct_tau[:, 0],
                 "time_constant": ct_tau[:, 1], "mounts": mounts}
        if name not in table:
            raise AttributeError(name)
        return table[name]

    def write_row(self, i, cfg: VehicleConfig):
        """Give env ``i`` the parameters of ``cfg`` (same actuator layout), as a new hull type."""
        self._st._assign_vehicle(int(i), cfg)


class BatchState:
    """N environments of one vehicle (or a mixed fleet) resident in HBM."""

    def __init__(self, vehicles, counts, sim: SimConfig, master_seed=0, device=None,
                 dtype=torch.float32, env_offset=0, rng="philox"):
        if dtype not in (torch.float32, torch.float64):
            raise EngineError("dtype must be torch.float32 or torch.float64")
        if rng not in RNG_GENERATORS:
            raise EngineError(f"rng must be one of {sorted(RNG_GENERATORS)}, got {rng!r}")
        self.rng = rng
        self.sim = sim
        self.vehicles = list(vehicles)
        self.vehicle = self.vehicles[0]
        self.master_seed = int(master_seed)
        self.env_offset = int(env_offset)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.dtype = dtype
        n = int(sum(counts))
        if n != sim.batch_size:
            raise EngineError(f"fleet counts sum to {n}, batch_size is {sim.batch_size}")
        self.n_envs = n
        self.a_max = max(v.action_dim for v in self.vehicles)
        self._ld = ld = max(_ALIGN, -(-n // _ALIGN) * _ALIGN)
        kw = dict(device=self.device)
        # one SoA block: rows 0-2 p, 3-6 q, 7-12 nu, 13.. act (p/q/nu are one
        # contiguous [13][ld] span, so a host snapshot of the pose is one copy)
        self._soa = torch.zeros((13 + self.a_max, ld), dtype=dtype, **kw)
        self._p, self._q = self._soa[0:3], self._soa[3:7]
        self._nu, self._act = self._soa[7:13], self._soa[13:]
        self._q[0] = 1.0
        self._cur = None
        self._cs = None
        self.steps = torch.zeros(ld, dtype=torch.int32, **kw)[:n]
        self.episodes = torch.full((ld,), -1, dtype=torch.int32, **kw)[:n]
        self.diverged = torch.zeros(ld, dtype=torch.bool, **kw)[:n]
        self._type = None
        self._runs = None  # contiguous per-type runs [(type, first row)] of a fleet batch
        if len(self.vehicles) > 1:
            ids = np.repeat(np.arange(len(counts), dtype=np.uint8), counts)
            self._type = torch.zeros(ld, dtype=torch.uint8, **kw)
            self._type[:n] = torch.from_numpy(ids).to(self.device)
            starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(int)
            self._runs = [(t, int(s0)) for t, (s0, c) in enumerate(zip(starts, counts)) if c > 0]
        self._ov = None
        self._ov_keys = None
        self._payload_offsets = False  # some env may carry a payload off the origin
        self._server = None  # active `serve` context (resident step kernel)
        self._pin = None  # pinned staging for host-side commands (step_batch host path)
        self._dcmd = None
        self._pinned_cache = {}
        self._slots = {}
        self._host_overlays = {}
        self._hulls = [pack_hull(v) for v in self.vehicles]
        self._ctx = C.c_void_p()
        arr = (N.Hull * len(self._hulls))(*self._hulls)
        N.check(N.load().uuv_ctx_create(arr, len(self._hulls), C.byref(self._ctx)), EngineError)
        self.params = ParamsView(self)
        self.layout = _Layout(self)

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and ctx.value:
            try:
                N.load().uuv_ctx_destroy(ctx)
            except Exception:
                pass

    # ---------------------------------------------------------------- reference fields
    @property
    def p(self):
        return self._p[:, :self.n_envs].t()

    @property
    def q(self):
        return self._q[:, :self.n_envs].t()

    @property
    def nu(self):
        return self._nu[:, :self.n_envs].t()

    @property
    def act(self):
        return self._act[:, :self.n_envs].t()

    @property
    def current_ned(self):
        """(N,3) NED current.  Touching it enables the current term in the kernel."""
        self._enable_current()
        return self._cur[:, :self.n_envs].t()

    @property
    def type_id(self):
        return None if self._type is None else self._type[:self.n_envs]

    @property
    def tilt(self):
        """Tilt angles stay at their defaults (engine.py:139-143, 507)."""
        cols = [[a.tilt_angle_default for a in v.actuators] + [0.0] * (self.a_max - v.action_dim)
                for v in self.vehicles]
        t = torch.tensor(cols, dtype=self.dtype, device=self.device)
        ids = self.type_id.long() if self._type is not None else torch.zeros(
            self.n_envs, dtype=torch.long, device=self.device)
        return t[ids]

    @property
    def overlays(self) -> list:
        """Per-env overlay dicts of the last reset (copied to the host)."""
        n = self.n_envs
        out = [dict(self._host_overlays.get(i, {})) for i in range(n)]
        if self._ov is None:
            return out
        ov = self._ov[:, :n].cpu().numpy()
        keys = self._ov_keys[:n].cpu().numpy().astype(np.int64) & 0xFFFF
        for i in range(n):
            if i in self._host_overlays or keys[i] == 0:
                continue
            d = {}
            for name, s0 in self._slots.items():
                if keys[i] >> N.OV_INDEX[name] & 1:
                    if name == "payload_position":
                        d[name] = ov[s0:s0 + 3, i].copy()
                    elif name == "mount_position_jitter":
                        d[name] = ov[s0:s0 + 3, i].copy()
                    else:
                        d[name] = float(ov[s0, i])
            out[i] = d
        return out

    def env_rng(self, i: int) -> np.random.Generator:
        """The counter-based substream of env i's current episode (engine.py:291-295)."""
        return RNG_GENERATORS[self.rng](self.master_seed, self.env_offset + int(i),
                                        int(self.episodes[int(i)].item()))

    # ---------------------------------------------------------------- internals
    def _stream(self):
        return _raw_stream(self._dev_index)

    def _enable_current(self):
        if self._cur is None:
            self._cur = torch.zeros((3, self._ld), dtype=self.dtype, device=self.device)
            self._cs = None

    def _ensure_slots(self, keys):
        keys = [k for k in keys if k in N.OV_INDEX]
        missing = [k for k in keys if k not in self._slots]
        if not missing:
            return
        names = sorted(set(self._slots) | set(missing), key=lambda k: N.OV_INDEX[k])
        slots, n_slots = {}, 0
        for k in names:
            slots[k] = n_slots
            n_slots += N.OV_WIDTH[k]
        ov = torch.empty((n_slots, self._ld), dtype=torch.float64, device=self.device)
        for k in names:
            s0, w = slots[k], N.OV_WIDTH[k]
            if k in self._slots:
                o0 = self._slots[k]
                ov[s0:s0 + w] = self._ov[o0:o0 + w]
            else:
                ov[s0:s0 + w] = N.OV_IDENTITY[k]
        self._ov, self._slots = ov, slots
        self._cs = None
        if self._ov_keys is None:
            self._ov_keys = torch.zeros(self._ld, dtype=torch.int16, device=self.device)

    def _cstate(self) -> N.State:
        if self._cs is None:
            self._cs = self._build_cstate()
        return self._cs

    def _build_cstate(self) -> N.State:
        s = N.State()
        # the reference's state fields cross the ABI as DLPack tensors; the C side
        # validates dtype, device, shapes and the SoA strides and fills the pointers
        n = self.n_envs
        fields = [N.dl(self.p), N.dl(self.q), N.dl(self.nu), N.dl(self.act),
                  N.dl(self._cur[:, :n].t()) if self._cur is not None else None,
                  N.dl(self.steps), N.dl(self.episodes), N.dl(self.diverged)]
        ptrs = (C.c_void_p * N.DL_COUNT)(*[N.dl_ptr(f) for f in fields])
        N.check(N.load().uuv_state_from_dlpack(C.byref(s), ptrs, N.DL_COUNT), EngineError)
        s.env_offset = self.env_offset
        s.type_id = self._type.data_ptr() if self._type is not None else None
        s.overlay = self._ov.data_ptr() if self._ov is not None else None
        s.overlay_keys = self._ov_keys.data_ptr() if self._ov_keys is not None else None
        s.n_slots = 0 if self._ov is None else self._ov.shape[0]
        for k in range(N.OV_COUNT):
            s.slot[k] = -1
        for name, s0 in self._slots.items():
            s.slot[N.OV_INDEX[name]] = s0
        s.flags = 0 if self._payload_offsets else N.STATE_PAYLOAD_AT_ORIGIN
        runs = self._runs if self._runs is not None and len(self._runs) <= N.MAX_RUNS else []
        s.n_runs = len(runs)
        for r, (t, s0) in enumerate(runs):
            s.run_type[r], s.run_start[r] = t, s0
        return s

    def _note_sampler(self, sampler: "DeviceSampler"):
        """Record what a device sampler can write (slots, current, payload offsets)."""
        keys = sampler.keys()
        if keys:
            self._ensure_slots(keys)
        if sampler.current_spec:
            self._enable_current()
        p = (sampler.overlay_spec or {}).get("payload_position")
        if p is not None and p.distribution.support() != (0.0, 0.0):
            self._payload_offsets = True
            self._cs = None

    def _assign_vehicle(self, i, cfg):
        if cfg.action_dim > self.a_max:
            raise EngineError("write_row: vehicle has more actuators than the batch")
        for t, v in enumerate(self.vehicles):
            if v is cfg:
                break
        else:
            if len(self.vehicles) >= N.MAX_TYPES:
                raise EngineError(f"write_row: at most {N.MAX_TYPES} distinct parameter sets "
                                  "per batch in the device build")
            self.vehicles.append(cfg)
            self._hulls.append(pack_hull(cfg))
            t = len(self.vehicles) - 1
            arr = (N.Hull * len(self._hulls))(*self._hulls)
            N.check(N.load().uuv_ctx_set_hulls(self._ctx, arr, len(self._hulls)), EngineError)
        if self._type is None:
            self._type = torch.zeros(self._ld, dtype=torch.uint8, device=self.device)
        self._type[i] = t
        self._runs = None  # rows of a type are no longer known to be contiguous
        self._cs = None


class _Layout:
    def __init__(self, st: BatchState):
        self.action_dim = st.vehicle.action_dim
        self.a_max = st.a_max
        self.fluid_density = st.vehicle.coeffs.fluid_density
        self.gravity = st.vehicle.coeffs.gravity


# ================================================================ public API


def make_batch(vehicle: VehicleConfig, sim: SimConfig, master_seed: int = 0, *, device=None,
               dtype=torch.float32, env_offset: int = 0, rng: str = "philox") -> BatchState:
    """Allocate a batch primed with the base vehicle; call reset_envs to start.

    ``rng``: ``"philox"`` (default) or ``"pcg64"`` — the reference's own
    PCG64/SeedSequence streams, for resets bit-identical to the unmodified reference.
    """
    return BatchState([vehicle], [sim.batch_size], sim, master_seed, device, dtype, env_offset,
                      rng)


def make_fleet_batch(vehicles, counts, sim: SimConfig, master_seed: int = 0, *, device=None,
                     dtype=torch.float32, env_offset: int = 0, rng: str = "philox") -> BatchState:
    """Mixed-vehicle batch: contiguous env blocks per vehicle type, commands padded to A_max."""
    if len(vehicles) != len(counts) or not 1 <= len(vehicles) <= N.MAX_TYPES:
        raise EngineError(f"need 1..{N.MAX_TYPES} vehicles with one count each")
    return BatchState(vehicles, counts, sim, master_seed, device, dtype, env_offset, rng)


def _commands(state: BatchState, commands, width):
    n = state.n_envs
    if torch.is_tensor(commands):
        t = commands
        if tuple(t.shape) != (n, width):
            raise EngineError(f"commands: expected shape {(n, width)}, got {tuple(t.shape)}")
        if t.device != state.device or t.dtype != state.dtype:
            t = t.to(device=state.device, dtype=state.dtype)
    else:
        arr = np.asarray(commands, dtype=np.float64)
        if arr.shape != (n, width):
            raise EngineError(f"commands: expected shape {(n, width)}, got {arr.shape}")
        t = torch.from_numpy(arr).to(device=state.device, dtype=state.dtype)
    if t.stride(1) != 1 or t.stride(0) < width:
        t = t.contiguous()
    return t


def _cmd_width(state: BatchState) -> int:
    return state.a_max if len(state.vehicles) > 1 or state._type is not None else \
        state.vehicle.action_dim


class no_gc:
    """Keep Python's cyclic garbage collector off while a CUDA graph is captured: a
    collection inside the capture may free an older graph or stream (a previous
    env's episode loop, say), and destroying one is a prohibited call that
    invalidates the capture in progress."""

    def __enter__(self):
        import gc

        self._was = gc.isenabled()
        gc.disable()
        return self

    def __exit__(self, *exc):
        import gc

        if self._was:
            gc.enable()
        return False


class HostStepOut:
    """Pinned host buffers for one step's result (``uuv_host_out``): every field the
    reference's ``step_batch`` mutates in place (engine.py:418, 444-449).

    ``p`` (N,3), ``q`` (N,4), ``nu`` (N,6), ``act`` (N,A) are transposed views of
    row-major ``pose`` (13, N) / ``act_rows`` (A, N) buffers in the batch dtype;
    ``steps`` (N,) int32 and ``diverged`` (N,) bool.  ``fields`` selects what is
    returned (others stay None and are not transferred).
    """

    FIELDS = ("pose", "act", "steps", "diverged")

    def __init__(self, state: "BatchState", fields=FIELDS):
        bad = set(fields) - set(self.FIELDS)
        if bad:
            raise EngineError(f"HostStepOut: unknown fields {sorted(bad)}")
        n, w = state.n_envs, _cmd_width(state)
        self.n_envs, self.width, self.dtype = n, w, state.dtype

        def pinned(shape, dt):
            return torch.zeros(shape, dtype=dt).pin_memory()

        self.pose = pinned((13, n), state.dtype) if "pose" in fields else None
        self.act_rows = pinned((w, n), state.dtype) if "act" in fields else None
        self.steps = pinned((n,), torch.int32) if "steps" in fields else None
        self.diverged = pinned((n,), torch.bool) if "diverged" in fields else None
        self._c = N.HostOut(*[t.data_ptr() if t is not None else None
                              for t in (self.pose, self.act_rows, self.steps, self.diverged)])

    @property
    def p(self):
        return self.pose[0:3].t()

    @property
    def q(self):
        return self.pose[3:7].t()

    @property
    def nu(self):
        return self.pose[7:13].t()

    @property
    def act(self):
        return self.act_rows.t()

    @property
    def nbytes(self) -> int:
        """Bytes one step moves device -> host into these buffers."""
        return sum(t.numel() * t.element_size() for t in
                   (self.pose, self.act_rows, self.steps, self.diverged) if t is not None)


def _host_out(state: BatchState, pose_out, out):
    """The uuv_host_out of a step call (None when nothing is returned)."""
    if out is not None:
        if pose_out is not None:
            raise EngineError("pass either pose_out or out, not both")
        if not isinstance(out, HostStepOut):
            raise EngineError("out: expected an engine.HostStepOut")
        if (out.n_envs, out.width, out.dtype) != (state.n_envs, _cmd_width(state), state.dtype):
            raise EngineError(f"out: buffers for {out.n_envs} envs x {out.width} actuators "
                              f"({out.dtype}), batch has {state.n_envs} x {_cmd_width(state)} "
                              f"({state.dtype})")
        return out._c
    if pose_out is None:
        return None
    if not _pinned_ok(state, pose_out, (13, state.n_envs)):
        raise EngineError(f"pose_out: expected a pinned contiguous (13, {state.n_envs}) "
                          f"{state.dtype} tensor")
    return N.HostOut(pose_out.data_ptr(), None, None, None)


def step_batch(state: BatchState, commands, *, pose_out=None, out=None) -> BatchState:
    """Advance every environment one control step (engine.py:465-484).

    ``commands``: (N, A) CUDA tensor (one launch, no host sync), or host data — a CPU
    tensor or numpy array, staged through a pinned buffer and copied asynchronously.
    ``out``: a ``HostStepOut`` receiving the step's result in host memory (p, q, nu,
    act, steps, diverged — what the reference's in-place step leaves in its numpy
    state); the call waits for it.  ``pose_out``: shorthand for the pose rows only,
    a pinned CPU tensor (13, N) in the batch dtype (rows p (3), q (4), nu (6)).
    """
    if state._server is not None:
        return state._server.step(commands, pose_out, out)
    width = _cmd_width(state)
    if pose_out is not None or out is not None or not isinstance(commands, torch.Tensor) \
            or not commands.is_cuda:
        return _step_host(state, commands, width, _host_out(state, pose_out, out))
    cmd = _commands(state, commands, width)
    arg = N.DLArg(cmd)
    status = N.load().uuv_step_dl(state._ctx, C.byref(state._cstate()), arg,
                                  state.sim.substeps, state.sim.dt, state._stream())
    if status:
        N.check(status, EngineError)
    return state


def rollout(state: BatchState, commands, steps: int | None = None, *, start: int = 0,
            trace=None, ready=None, out=None) -> BatchState:
    """``steps`` control steps in ONE kernel launch, the state held in registers
    throughout (``uuv_rollout_dl``): bit for bit

        for t in range(steps):
            step_batch(state, commands[(start + t) % S])

    ``commands``: (S, N, A) -- a ring of S command slots -- or (N, A), held for every
    step (the ``throughput_probe`` protocol, engine.py:541-564); ``steps`` defaults to
    S.  ``trace``: optional (>= steps, 13, N) tensor of the batch dtype receiving p (3),
    q (4), nu (6) after every step, or (>= steps, 13 + A, N) receiving act (A) too.
    Both are CUDA tensors, or pinned host tensors: the kernel then reads the command
    rows over the host link (one step ahead) and writes the trace rows into host
    memory as it produces them -- a host-to-host rollout in one launch, and the call
    returns once the launch has finished (the host buffers are then free to reuse).
    ``out``: a ``HostStepOut`` receiving the result after the last step (as
    ``step_batch(..., out=)``), written into its pinned rows by the kernel; the call
    waits for it.
    ``ready``: optional int32 CUDA counter; step t waits until ``ready > t`` -- a
    producer on another stream writes slot t and then raises the counter (a
    device-side command ring).  The producer's kernels must already be loaded (under
    CUDA lazy loading a first launch waits for the device, i.e. for the waiting
    rollout); a rollout that sees no new slot for 10 s stops instead of hanging.
    """
    if state._server is not None:
        raise EngineError("rollout: the batch is being served (leave the serve() block first)")
    n, w = state.n_envs, _cmd_width(state)
    if not torch.is_tensor(commands):
        raise EngineError("commands: rollout takes a CUDA or pinned host tensor (S, N, A) "
                          "or (N, A)")
    cmd = commands if commands.dim() == 3 else commands.unsqueeze(0)
    if cmd.dim() != 3 or tuple(cmd.shape[1:]) != (n, w):
        raise EngineError(f"commands: expected shape (S, {n}, {w}) or ({n}, {w}), "
                          f"got {tuple(commands.shape)}")
    host = not cmd.is_cuda
    if host:
        if not (cmd.dtype == state.dtype and cmd.is_contiguous() and _is_pinned(state, cmd)):
            raise EngineError(f"commands: host commands must be a pinned contiguous "
                              f"{state.dtype} tensor")
    else:
        if cmd.dtype != state.dtype or cmd.device != state.device:
            cmd = cmd.to(device=state.device, dtype=state.dtype)
        if cmd.stride(2) != 1:
            cmd = cmd.contiguous()
    if trace is not None and not trace.is_cuda:
        if not (trace.is_contiguous() and _is_pinned(state, trace)):
            raise EngineError("trace: a host trace must be a pinned contiguous tensor")
        host = True
    ho = _host_out(state, None, out)
    steps = cmd.shape[0] if steps is None else int(steps)
    if steps < 0 or start < 0:
        raise EngineError("steps and start must be >= 0")
    args = [N.DLArg(cmd), N.dl(trace), N.dl(ready)]
    status = N.load().uuv_rollout_dl(state._ctx, C.byref(state._cstate()), args[0], int(start),
                                     steps, state.sim.substeps, state.sim.dt, args[1], args[2],
                                     None if ho is None else C.byref(ho), state._stream())
    if status:
        N.check(status, EngineError)
    if host or out is not None:  # the kernel reads / writes host buffers until it ends
        torch.cuda.current_stream(state.device).synchronize()
    return state


class serve:
    """Host-in-the-loop stepping through a resident step kernel (``uuv_server_*``).

        with serve(state):
            for t in range(T):
                step_batch(state, pinned_cmds[t], pose_out=pinned_pose)

    Inside the block ``step_batch`` takes host commands (pinned tensors, or any
    host array staged through a pinned buffer) and optionally a pinned (13, N)
    ``pose_out``; each call rings a doorbell in mapped pinned memory and returns
    when every env has stepped and its pose rows have landed -- no kernel
    launch and no stream synchronisation per step.  Results are bit-identical to
    ``step_batch`` outside the block.  The kernel owns the state while it runs:
    other operations on the batch raise until the block exits, and a
    device-wide synchronisation (``torch.cuda.synchronize()``) would wait for
    the kernel -- use stream-level synchronisation inside the block.  It stops
    by itself after ``idle_timeout_ms`` without a step.
    """

    def __init__(self, state: "BatchState", idle_timeout_ms: int = 10_000):
        self.state = state
        self.idle_timeout_ms = int(idle_timeout_ms)
        self._h = None

    def __enter__(self):
        st = self.state
        if st._server is not None:
            raise EngineError("serve: this batch already has a step server")
        h = C.c_void_p()
        N.check(N.load().uuv_server_start(st._ctx, C.byref(st._cstate()), st.sim.substeps,
                                          st.sim.dt, st._stream(), self.idle_timeout_ms,
                                          C.byref(h)), EngineError)
        self._h = h
        self._width = _cmd_width(st)
        st._server = self
        return self

    def step(self, commands, pose_out=None, out=None):
        st = self.state
        n, width = st.n_envs, self._width
        if isinstance(commands, torch.Tensor) and commands.device.type == "cpu" and \
                _pinned_ok(st, commands, (n, width)):
            src = commands
        elif isinstance(commands, torch.Tensor) and commands.is_cuda:
            raise EngineError("commands: inside serve() pass host commands (pinned tensor or "
                              "array), not a CUDA tensor")
        else:
            arr = np.asarray(commands.cpu() if isinstance(commands, torch.Tensor) else commands)
            if arr.shape != (n, width):
                raise EngineError(f"commands: expected shape {(n, width)}, got {arr.shape}")
            if st._pin is None:
                st._pin = torch.empty((n, width), dtype=st.dtype).pin_memory()
            st._pin.numpy()[...] = arr
            src = st._pin
        ho = _host_out(st, pose_out, out)
        status = N.load().uuv_server_step(self._h, src.data_ptr(), width,
                                          C.byref(ho) if ho is not None else None)
        if status:
            N.check(status, EngineError)
        return st

    def __exit__(self, *exc):
        st = self.state
        st._server = None
        status = N.load().uuv_server_stop(self._h)
        self._h = None
        N.check(status, EngineError)
        return False


def _is_pinned(state: BatchState, t) -> bool:
    """``t.is_pinned()``, cached per tensor object like ``_pinned_ok``."""
    return _pinned_ok(state, t, tuple(t.shape), dtype=t.dtype)


def _pinned_ok(state: BatchState, t, shape, dtype=None) -> bool:
    """Pinned, contiguous, batch dtype and shape.  Cached per tensor object (a weak
    reference plus its data address), so a freed buffer whose address is reused
    is checked afresh."""
    key = id(t)
    hit = state._pinned_cache.get(key)
    if hit is not None and hit[0]() is t and hit[1] == t.data_ptr():
        return hit[2]
    ok = (tuple(t.shape) == shape and t.dtype == (state.dtype if dtype is None else dtype)
          and t.is_contiguous() and t.is_pinned())
    if len(state._pinned_cache) > 64:
        state._pinned_cache.clear()
    state._pinned_cache[key] = (weakref.ref(t), t.data_ptr(), ok)
    return ok


def _step_host(state: BatchState, commands, width, ho):
    n = state.n_envs
    st = state
    if st._pin is None:
        st._pin = torch.empty((n, width), dtype=st.dtype).pin_memory()
        st._dcmd = torch.empty((n, width), dtype=st.dtype, device=st.device)
    src = None
    if isinstance(commands, torch.Tensor):
        if commands.device.type == "cpu":
            if _pinned_ok(st, commands, (n, width)):
                src = commands
            else:
                if tuple(commands.shape) != (n, width):
                    raise EngineError(f"commands: expected shape {(n, width)}, "
                                      f"got {tuple(commands.shape)}")
                st._pin.copy_(commands)
                src = st._pin
    else:
        arr = np.asarray(commands)
        if arr.shape != (n, width):
            raise EngineError(f"commands: expected shape {(n, width)}, got {arr.shape}")
        st._pin.numpy()[...] = arr
        src = st._pin
    lib = N.load()
    if src is None:  # device commands with host result rows
        cmd = _commands(state, commands, width)
        N.check(lib.uuv_step_dl(st._ctx, C.byref(st._cstate()), N.DLArg(cmd),
                                st.sim.substeps, st.sim.dt, st._stream()), EngineError)
        torch.cuda.current_stream(st.device).synchronize()
        _copy_result(st, ho)
        return state
    status = lib.uuv_step_host(st._ctx, C.byref(st._cstate()), src.data_ptr(), width,
                               st._dcmd.data_ptr(), C.byref(ho) if ho is not None else None,
                               st.sim.substeps, st.sim.dt, st._stream(),
                               1 if ho is not None or src is st._pin else 0)
    if status:
        N.check(status, EngineError)
    return state


def _copy_result(st: BatchState, ho):
    """Synchronous copy of the state into the host result rows (device commands path)."""
    if ho is None:
        return
    n, w = st.n_envs, _cmd_width(st)

    def into(addr, src):
        if addr:  # the caller's pinned buffer at `addr`, viewed as a tensor
            buf = (C.c_char * (src.numel() * src.element_size())).from_address(addr)
            torch.frombuffer(buf, dtype=src.dtype).view(src.shape).copy_(src)

    into(ho.pose, st._soa[:13, :n].contiguous().cpu())
    into(ho.act, st._act[:w, :n].contiguous().cpu())
    into(ho.steps, st.steps.cpu())
    into(ho.diverged, st.diverged.cpu())


def _mask(state: BatchState, mask):
    n = state.n_envs
    if torch.is_tensor(mask):
        m = mask
        if tuple(m.shape) != (n,):
            raise EngineError(f"mask: expected shape {(n,)}, got {tuple(m.shape)}")
        return m.to(device=state.device, dtype=torch.bool).contiguous()
    arr = np.asarray(mask, dtype=bool)
    if arr.shape != (n,):
        raise EngineError(f"mask: expected shape {(n,)}, got {arr.shape}")
    return torch.from_numpy(arr).to(state.device)


def reset_envs(state: BatchState, mask, sampler: InitSampler = default_sampler) -> BatchState:
    """Re-initialise masked envs from their episode substreams (engine.py:487-512).

    ``default_sampler`` and ``DeviceSampler`` objects run in the reset kernel;
    any other Python callable runs on the host, one call per masked row, with
    the same Philox stream, and the rows are uploaded.
    """
    if state._server is not None:
        raise EngineError("reset_envs: the batch is being served (leave the serve() block first)")
    m = _mask(state, mask)
    if sampler is default_sampler:
        sampler = _IDENTITY
    if isinstance(sampler, DeviceSampler):
        _device_reset(state, m, sampler)
    else:
        _host_reset(state, m, sampler)
    return state


def _device_reset(state: BatchState, m, sampler: DeviceSampler):
    state._note_sampler(sampler)
    packed = sampler.pack()
    packed.rng_mode = N.RNG_MODES[state.rng]
    if state._host_overlays:
        idx = torch.nonzero(m).flatten().cpu().tolist()
        for i in idx:
            state._host_overlays.pop(i, None)
    N.check(N.load().uuv_reset_dl(state._ctx, C.byref(state._cstate()), N.DLArg(m),
                                  C.byref(packed), state.master_seed & M64, state._stream()),
            EngineError)


def _host_reset(state: BatchState, m, sampler):
    rows = torch.nonzero(m).flatten().cpu().numpy()
    if rows.size == 0:
        return
    eps = state.episodes[torch.from_numpy(rows).to(state.device)].cpu().numpy().astype(np.int64) + 1
    inits = []
    for i, ep in zip(rows, eps):
        init = sampler(int(i), int(ep), RNG_GENERATORS[state.rng](
            state.master_seed, state.env_offset + int(i), int(ep)))
        ov = dict(init.overlay)
        if ov:
            validate_overlay(state.vehicles[0] if state._type is None else state.vehicle, ov)
        inits.append((init, ov))
    keys = sorted({k for _, ov in inits for k in ov if k in N.OV_INDEX})
    if keys:
        state._ensure_slots(keys)
    cur = np.array([np.asarray(init.current_ned, float) for init, _ in inits])
    if np.any(cur != 0.0):
        state._enable_current()
    dev = state.device
    idx = torch.from_numpy(rows).to(dev)
    dt = state.dtype
    p = torch.from_numpy(np.array([init.pose.p for init, _ in inits], float)).to(dev, dt)
    q = torch.from_numpy(np.array([init.pose.q for init, _ in inits], float)).to(dev, dt)
    nu = torch.from_numpy(np.array([np.asarray(init.nu, float) for init, _ in inits])).to(dev, dt)
    state._p[:, idx] = p.t()
    state._q[:, idx] = q.t()
    state._nu[:, idx] = nu.t()
    state._act[:, idx] = 0.0
    if state._cur is not None:
        state._cur[:, idx] = torch.from_numpy(cur).to(dev, dt).t()
    state.steps[idx] = 0
    state.diverged[idx] = False
    state.episodes[idx] = torch.from_numpy(eps.astype(np.int32)).to(dev)
    if state._ov is not None:
        block = np.empty((state._ov.shape[0], rows.size))
        kbits = np.zeros(rows.size, dtype=np.int64)
        for name, s0 in state._slots.items():
            block[s0:s0 + N.OV_WIDTH[name]] = N.OV_IDENTITY[name]
        for r, (_, ov) in enumerate(inits):
            for name, v in ov.items():
                if name not in state._slots:
                    continue
                s0 = state._slots[name]
                kbits[r] |= 1 << N.OV_INDEX[name]
                if name == "payload_position":
                    block[s0:s0 + 3, r] = np.asarray(v, float)
                    if np.any(block[s0:s0 + 3, r] != 0.0):
                        state._payload_offsets = True
                        state._cs = None
                elif name == "mount_position_jitter":
                    jv = np.asarray(v, float)
                    jm = np.zeros((N.MAX_ACT, 3))
                    jm[:] = jv if jv.ndim == 1 else 0.0
                    if jv.ndim == 2:
                        jm[:jv.shape[0]] = jv
                    block[s0:s0 + 3 * N.MAX_ACT, r] = jm.ravel()
                else:
                    block[s0, r] = float(v)
        state._ov[:, idx] = torch.from_numpy(block).to(dev)
        state._ov_keys[idx] = torch.from_numpy(kbits.astype(np.int16)).to(dev)
    for r, i in enumerate(rows):
        state._host_overlays[int(i)] = inits[r][1]


def env_snapshot(state: BatchState, i: int) -> dict:
    """One env's state and reset context as host copies (engine.py:515-527)."""
    i = int(i)
    snap = {
        "p": state.p[i].double().cpu().numpy().copy(),
        "q": state.q[i].double().cpu().numpy().copy(),
        "nu": state.nu[i].double().cpu().numpy().copy(),
        "act": state.act[i, :state.vehicles[0].action_dim if state._type is None else
                         state.a_max].double().cpu().numpy().copy(),
        "current_ned": (state._cur[:, i].double().cpu().numpy().copy()
                        if state._cur is not None else np.zeros(3)),
        "steps": int(state.steps[i].item()),
        "episode": int(state.episodes[i].item()),
        "diverged": bool(state.diverged[i].item()),
        "overlay": dict(state.overlays[i]),
    }
    return snap


def current_in_body(q, current_ned):
    """Irrotational current as a body-frame 6-vector (engine.py:329-332), torch."""
    q = torch.as_tensor(q)
    c = torch.as_tensor(current_ned, dtype=q.dtype, device=q.device)
    w, u = q[..., :1], -q[..., 1:]
    uv = torch.linalg.cross(u, c.expand_as(u))
    lin = c + 2.0 * (w * uv + torch.linalg.cross(u, uv))
    return torch.cat([lin, torch.zeros_like(lin)], dim=-1)


@dataclass
class ThroughputReport:
    batch_size: int
    workers: int
    n_steps: int
    elapsed_s: float
    aggregate_steps_per_s: float
    per_env_steps_per_s: float
    diverged_envs: int = 0


def throughput_probe(sim: SimConfig, vehicle: VehicleConfig, duration: float = 2.0,
                     warmup_steps: int = 20, seed: int = 0, *, dtype=torch.float32,
                     device=None, mode: str = "rollout") -> ThroughputReport:
    """Stepping rate with active rotors (engine.py:541-564), device-timed.

    Commands are ``default_rng(seed).uniform(-1, 1, (N, A))`` held fixed, as in
    the reference.  ``mode``: ``"rollout"`` runs chunks of 100 steps as one
    ``rollout`` launch each (the state held in registers, bit for bit 100
    ``step_batch`` calls); ``"graph"`` replays a captured CUDA graph of 100
    ``step_batch`` launches; ``"launch"`` launches every step from Python.
    Timed with CUDA events.
    """
    if mode not in ("rollout", "graph", "launch"):
        raise EngineError(f"mode must be rollout, graph or launch, got {mode!r}")
    st = make_batch(vehicle, sim, master_seed=seed, device=device, dtype=dtype)
    reset_envs(st, np.ones(sim.batch_size, bool))
    cmds = torch.from_numpy(np.random.default_rng(seed).uniform(
        -1.0, 1.0, size=(sim.batch_size, vehicle.action_dim))).to(st.device, dtype)
    for _ in range(warmup_steps):
        step_batch(st, cmds)
    chunk = 100
    if mode == "rollout":
        def run():
            rollout(st, cmds, chunk)
    elif mode == "graph":
        s = torch.cuda.Stream(st.device)
        s.wait_stream(torch.cuda.current_stream(st.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            step_batch(st, cmds)
            with torch.cuda.graph(g, stream=s), no_gc():
                for _ in range(chunk):
                    step_batch(st, cmds)
        torch.cuda.current_stream(st.device).wait_stream(s)
        run = g.replay
    else:
        def run():
            for _ in range(chunk):
                step_batch(st, cmds)
    torch.cuda.synchronize(st.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_steps, t_wall = 0, time.perf_counter()
    e0.record()
    while True:
        run()
        n_steps += chunk
        if time.perf_counter() - t_wall >= duration:
            break
    e1.record()
    torch.cuda.synchronize(st.device)
    el = e0.elapsed_time(e1) / 1e3
    return ThroughputReport(batch_size=sim.batch_size, workers=sim.workers, n_steps=n_steps,
                            elapsed_s=el, aggregate_steps_per_s=sim.batch_size * n_steps / el,
                            per_env_steps_per_s=n_steps / el,
                            diverged_envs=int(st.diverged.sum().item()))


def substep_terms(state: BatchState, commands) -> dict:
    """First-substep intermediates (tau, w_hydro, C_RB nu, nudot, next state) without
    advancing the batch — the quantities engine.py:425-433 forms; for parity checks."""
    width = state.a_max if state._type is not None else state.vehicle.action_dim
    cmd = _commands(state, commands, width)
    out = torch.empty((state.n_envs, 48), dtype=torch.float64, device=state.device)
    N.check(N.load().uuv_substep_terms(state._ctx, C.byref(state._cstate()), cmd.data_ptr(),
                                       cmd.stride(0), state.sim.dt / state.sim.substeps,
                                       out.data_ptr(), state._stream()), EngineError)
    A = width
    return {"tau": out[:, 0:6], "hydro": out[:, 6:12], "c_rb": out[:, 12:18],
            "acc": out[:, 18:24], "nu_new": out[:, 24:30], "p_new": out[:, 30:33],
            "q_new": out[:, 33:37], "act_new": out[:, 37:37 + A], "ok": out[:, 45] > 0.5}
