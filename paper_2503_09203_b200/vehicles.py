"""Vehicle parameter model (host side) for the B200 hydrodynamic step.

Mirrors the data model the reference engine consumes:

* ``RigidBodyParams`` / ``HydroCoeffs``  — ``uuvsim/hydrodynamics.py:48-85``
* ``ActuatorSpec`` / ``RudderGeometry`` / ``MLPWeights`` — ``uuvsim/actuation.py:34-131``
* ``VehicleConfig``, ``load_vehicle``, ``parse_vehicle`` (schema_version 1
  documents), ``apply_overlay``, ``compose_with_payload`` —
  ``uuvsim/vehicles/__init__.py:84-505``

These objects are plain host data: the device never sees them.  The engine
packs one ``VehicleConfig`` into a fixed-layout *hull table* (``pack_hull``)
that travels to the GPU by value inside the kernel parameter block, so every
per-vehicle constant is a constant-bank operand of the FFMA that uses it.
"""

from __future__ import annotations

import copy
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import fleet

SCHEMA_VERSION = 1
BUILTIN_VEHICLES = fleet.BUILTIN_VEHICLES

PROPELLER, RUDDER, TILTROTOR = "propeller", "rudder", "tiltrotor"
ZERO_ORDER, FIRST_ORDER, DATA_DRIVEN = "zero_order", "first_order", "data_driven"
KIND_CODE = {PROPELLER: 0, RUDDER: 1, TILTROTOR: 2}
MODEL_CODE = {ZERO_ORDER: 0, FIRST_ORDER: 1, DATA_DRIVEN: 2}

RATIO_KEYS = ("mass*", "volume*", "inertia*", "added_mass*", "damping*",
              "time_constant*", "thrust_coeff*")
SPECIAL_KEYS = ("cobm", "payload_mass*", "payload_position", "mount_position_jitter")
ENVIRONMENT_KEYS = ("current_velocity", "current_direction")
OVERLAY_KEYS = RATIO_KEYS + SPECIAL_KEYS + ENVIRONMENT_KEYS

GRAVITY = 9.81
FLUID_DENSITY = 1000.0


class ConfigError(ValueError):
    """Schema violation; message starts with the offending field path."""


class ParameterError(ValueError):
    """Physically invalid parameters (hydrodynamics.py:33)."""


class ActuatorError(ValueError):
    """Invalid actuator description (actuation.py:30)."""


def _require_spd(M, name, semi=False, tol=1e-9):
    """Symmetric (1e-8) and (semi-)definite check, hydrodynamics.py:37-45."""
    M = np.asarray(M, dtype=float)
    if not np.allclose(M, np.swapaxes(M, -1, -2), atol=1e-8):
        raise ParameterError(f"{name}: matrix must be symmetric")
    lam = np.linalg.eigvalsh(M)
    floor = -tol if semi else tol
    if np.any(lam < floor):
        what = "positive semi-definite" if semi else "positive definite"
        raise ParameterError(f"{name}: matrix must be {what} (min eigenvalue {lam.min():.3e})")


@dataclass
class RigidBodyParams:
    mass: float
    inertia: np.ndarray
    r_g: np.ndarray = field(default_factory=lambda: np.zeros(3))
    r_b: np.ndarray = field(default_factory=lambda: np.zeros(3))
    displaced_volume: float = 0.0

    def __post_init__(self):
        self.inertia = np.asarray(self.inertia, dtype=float)
        self.r_g = np.asarray(self.r_g, dtype=float)
        self.r_b = np.asarray(self.r_b, dtype=float)
        if not self.mass > 0:
            raise ParameterError(f"mass: must be > 0, got {self.mass}")
        if self.displaced_volume < 0:
            raise ParameterError(f"displaced_volume: must be >= 0, got {self.displaced_volume}")
        _require_spd(self.inertia, "inertia")


@dataclass
class HydroCoeffs:
    M_A: np.ndarray
    D_lin: np.ndarray
    D_quad: np.ndarray
    fluid_density: float = FLUID_DENSITY
    gravity: float = GRAVITY

    def __post_init__(self):
        self.M_A = np.asarray(self.M_A, dtype=float)
        self.D_lin = np.asarray(self.D_lin, dtype=float)
        self.D_quad = np.asarray(self.D_quad, dtype=float)
        for name in ("M_A", "D_lin", "D_quad"):
            _require_spd(getattr(self, name), name, semi=True)


@dataclass
class MLPWeights:
    """Rotor response net: (command, speed fraction) -> d(speed fraction)/dt."""

    layer_sizes: list
    weights: list
    biases: list
    activation: str = "tanh"

    def __post_init__(self):
        self.weights = [np.asarray(w, dtype=float) for w in self.weights]
        self.biases = [np.asarray(b, dtype=float) for b in self.biases]
        sz = list(self.layer_sizes)
        if len(self.weights) != len(sz) - 1 or len(self.biases) != len(sz) - 1:
            raise ActuatorError("weights/biases count must match layer_sizes")
        if sz[0] != 2 or sz[-1] != 1:
            raise ActuatorError("rotor MLP must map 2 inputs -> 1 output")
        for k, (w, b) in enumerate(zip(self.weights, self.biases)):
            if w.shape != (sz[k + 1], sz[k]):
                raise ActuatorError(f"weights[{k}]: expected shape {(sz[k + 1], sz[k])}, got {w.shape}")
            if b.shape != (sz[k + 1],):
                raise ActuatorError(f"biases[{k}]: expected shape {(sz[k + 1],)}")
        if self.activation not in ("tanh", "relu"):
            raise ActuatorError(f"unknown activation '{self.activation}'")


@dataclass
class RudderGeometry:
    area: float
    c_l_alpha: float
    c_d0: float = 0.02
    k_d: float = 1.0
    stall_angle: float = 0.52
    max_angle: float = 0.35
    fluid_density: float = 1000.0


@dataclass
class ActuatorSpec:
    index: int
    kind: str = PROPELLER
    mount_position: np.ndarray = field(default_factory=lambda: np.zeros(3))
    mount_axis: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0]))
    rotor_model: str = FIRST_ORDER
    time_constant: float = 0.15
    mlp: MLPWeights | None = None
    weights_ref: str | None = None
    thrust_coeff: float = 1e-4
    deadzone: float = 0.0
    max_speed: float = 400.0
    reaction_coeff: float = 0.0
    rudder: RudderGeometry | None = None
    tilt_range: float = 0.0
    tilt_axis: np.ndarray = field(default_factory=lambda: np.array([0.0, -1.0, 0.0]))
    tilt_angle_default: float = 0.0

    def __post_init__(self):
        self.mount_position = np.asarray(self.mount_position, dtype=float)
        ax = np.asarray(self.mount_axis, dtype=float)
        tk = np.asarray(self.tilt_axis, dtype=float)
        if np.linalg.norm(ax) < 1e-9:
            raise ActuatorError(f"actuator {self.index}: mount_axis must be nonzero")
        self.mount_axis = ax / np.linalg.norm(ax)
        self.tilt_axis = tk / np.linalg.norm(tk) if np.linalg.norm(tk) > 1e-9 else tk
        if self.kind not in KIND_CODE:
            raise ActuatorError(f"actuator {self.index}: unknown kind '{self.kind}'")
        if self.rotor_model not in MODEL_CODE:
            raise ActuatorError(f"actuator {self.index}: unknown rotor model '{self.rotor_model}'")
        if self.deadzone < 0:
            raise ActuatorError(f"actuator {self.index}: deadzone must be >= 0")
        if self.time_constant <= 0:
            raise ActuatorError(f"actuator {self.index}: time_constant must be > 0")
        if self.kind == RUDDER and self.rudder is None:
            raise ActuatorError(f"actuator {self.index}: rudder geometry missing")

    @property
    def state_limit(self) -> float:
        return self.rudder.max_angle if self.kind == RUDDER else self.max_speed


@dataclass
class Payload:
    mass: float
    attach_position: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.attach_position = np.asarray(self.attach_position, dtype=float)
        if self.mass < 0:
            raise ConfigError(f"payload.mass: must be >= 0, got {self.mass}")


@dataclass
class VehicleConfig:
    name: str
    rb: RigidBodyParams
    coeffs: HydroCoeffs
    actuators: list
    bounding_radius: float
    schema_version: int = SCHEMA_VERSION

    @property
    def action_dim(self) -> int:
        return len(self.actuators)


# ---------------------------------------------------------------- builders


def _mlp_from_dict(d) -> MLPWeights:
    return MLPWeights(layer_sizes=[int(s) for s in d["layer_sizes"]], weights=d["weights"],
                      biases=d["biases"], activation=d.get("activation", "tanh"))


def _from_fleet(name: str) -> VehicleConfig:
    entry = fleet.FLEET[name]
    h = entry["hull"]
    rb = RigidBodyParams(mass=h["mass"], inertia=np.diag(h["inertia_diag"]), r_g=h["r_g"],
                         r_b=h["r_b"], displaced_volume=h["volume"])
    co = HydroCoeffs(M_A=np.diag(h["added_mass_diag"]), D_lin=np.diag(h["linear_damping_diag"]),
                     D_quad=np.diag(h["quadratic_damping_diag"]),
                     fluid_density=h["fluid_density"], gravity=h["gravity"])
    acts = []
    for i, a in enumerate(entry["actuators"]):
        kw = dict(index=i, kind=a["kind"], mount_position=a["mount"], mount_axis=a["axis"],
                  rotor_model=a["model"], time_constant=a["time_constant"])
        if a["kind"] == RUDDER:
            kw["rudder"] = RudderGeometry(**a["rudder"])
        else:
            kw.update(thrust_coeff=a["thrust_coeff"], deadzone=a["deadzone"],
                      max_speed=a["max_speed"], reaction_coeff=a.get("reaction_coeff", 0.0))
        if a["kind"] == TILTROTOR:
            kw.update(tilt_range=a["tilt_range"], tilt_axis=a["tilt_axis"],
                      tilt_angle_default=a["tilt_default"])
        acts.append(ActuatorSpec(**kw))
    return VehicleConfig(name=name, rb=rb, coeffs=co, actuators=acts,
                         bounding_radius=entry["bounding_radius"])


def builtin_rotor_net(name: str) -> MLPWeights:
    return _mlp_from_dict(fleet.ROTOR_NETS[name])


# ---------------------------------------------------------------- schema v1 documents


def _field(doc, path, key, kind, required=True, default=None):
    where = f"{path}.{key}" if path else key
    if key not in doc:
        if required:
            raise ConfigError(f"{where}: missing required field")
        return default
    v = doc[key]
    ok = {
        float: lambda x: isinstance(x, (int, float)) and not isinstance(x, bool),
        int: lambda x: isinstance(x, int) and not isinstance(x, bool),
        str: lambda x: isinstance(x, str),
        list: lambda x: isinstance(x, list),
        dict: lambda x: isinstance(x, dict),
    }[kind]
    if not ok(v):
        label = {float: "a number", int: "an integer", str: "a string", list: "a list",
                 dict: "a mapping"}[kind]
        raise ConfigError(f"{where}: expected {label}, got {type(v).__name__}")
    return float(v) if kind is float else v


def _vec(doc, path, key, n, required=True, default=None):
    raw = _field(doc, path, key, list, required=required)
    if raw is None:
        return default
    where = f"{path}.{key}" if path else key
    try:
        v = np.asarray(raw, dtype=float)
    except (TypeError, ValueError):
        raise ConfigError(f"{where}: expected {n} numbers") from None
    if v.shape != (n,):
        raise ConfigError(f"{where}: expected {n} numbers, got shape {v.shape}")
    return v


def _square(doc, path, key, n):
    blk = _field(doc, path, key, dict)
    where = f"{path}.{key}"
    if "diag" in blk:
        return np.diag(_vec(blk, where, "diag", n))
    if "matrix" in blk:
        try:
            m = np.asarray(_field(blk, where, "matrix", list), dtype=float)
        except (TypeError, ValueError):
            raise ConfigError(f"{where}.matrix: expected a {n}x{n} matrix") from None
        if m.shape != (n, n):
            raise ConfigError(f"{where}.matrix: expected shape ({n}, {n}), got {m.shape}")
        return m
    raise ConfigError(f"{where}: expected 'diag' or 'matrix'")


def load_mlp_weights(path) -> MLPWeights:
    import yaml

    path = Path(path)
    try:
        doc = yaml.safe_load(path.read_text())
    except OSError as exc:
        raise ConfigError(f"weights file {path}: {exc}") from exc
    except yaml.YAMLError as exc:
        raise ConfigError(f"weights file {path}: invalid document ({exc})") from exc
    if not isinstance(doc, dict):
        raise ConfigError(f"weights file {path}: expected a mapping at top level")
    try:
        return MLPWeights(layer_sizes=[int(s) for s in _field(doc, "", "layer_sizes", list)],
                          weights=_field(doc, "", "weights", list),
                          biases=_field(doc, "", "biases", list),
                          activation=_field(doc, "", "activation", str, False, "tanh"))
    except (TypeError, ValueError) as exc:
        raise ConfigError(f"weights file {path}: {exc}") from exc


def _parse_actuator(doc, path, base_dir):
    idx = _field(doc, path, "index", int)
    kind = _field(doc, path, "kind", str)
    if kind not in KIND_CODE:
        raise ConfigError(f"{path}.kind: unknown actuator kind '{kind}'")
    mount = _vec(doc, path, "mount_position_m", 3)
    axis = _vec(doc, path, "mount_axis", 3)
    if abs(np.linalg.norm(axis) - 1.0) > 1e-6:
        raise ConfigError(f"{path}.mount_axis: must be a unit vector")
    model = _field(doc, path, "rotor_model", str)
    if model not in MODEL_CODE:
        raise ConfigError(f"{path}.rotor_model: unknown model '{model}'")
    kw = dict(index=idx, kind=kind, mount_position=mount, mount_axis=axis, rotor_model=model)
    if model == FIRST_ORDER:
        kw["time_constant"] = _field(doc, path, "time_constant_s", float)
        if kw["time_constant"] <= 0:
            raise ConfigError(f"{path}.time_constant_s: must be > 0")
    elif model == DATA_DRIVEN:
        ref = _field(doc, path, "weights_ref", str)
        wpath = Path(ref)
        if not wpath.is_absolute():
            if base_dir is None:
                raise ConfigError(f"{path}.weights_ref: relative path with no base directory")
            wpath = base_dir / wpath
        if wpath.exists():
            kw["mlp"] = load_mlp_weights(wpath)
        elif wpath.stem in fleet.ROTOR_NETS:  # builtin networks travel as source
            kw["mlp"] = builtin_rotor_net(wpath.stem)
        else:
            raise ConfigError(f"{path}.weights_ref: file not found: {wpath}")
        kw["weights_ref"] = ref
    if kind == RUDDER:
        r = _field(doc, path, "rudder", dict)
        rp = f"{path}.rudder"
        geom = RudderGeometry(
            area=_field(r, rp, "area_m2", float),
            c_l_alpha=_field(r, rp, "lift_slope_per_rad", float),
            c_d0=_field(r, rp, "drag_coeff_zero", float, False, 0.02),
            k_d=_field(r, rp, "drag_coeff_induced", float, False, 1.0),
            stall_angle=_field(r, rp, "stall_angle_rad", float, False, 0.52),
            max_angle=_field(r, rp, "max_angle_rad", float, False, 0.35),
            fluid_density=_field(r, rp, "fluid_density_kgm3", float, False, 1000.0))
        if geom.area <= 0:
            raise ConfigError(f"{rp}.area_m2: must be > 0")
        if geom.max_angle <= 0 or geom.stall_angle <= 0:
            raise ConfigError(f"{rp}: angle limits must be > 0")
        kw["rudder"] = geom
    else:
        kw["thrust_coeff"] = _field(doc, path, "thrust_coeff_ns2_per_rad2", float)
        kw["deadzone"] = _field(doc, path, "deadzone_rad_s", float, False, 0.0)
        kw["max_speed"] = _field(doc, path, "max_speed_rad_s", float)
        kw["reaction_coeff"] = _field(doc, path, "reaction_coeff_nms2_per_rad2", float, False, 0.0)
        if kw["max_speed"] <= 0:
            raise ConfigError(f"{path}.max_speed_rad_s: must be > 0")
        if kw["deadzone"] < 0:
            raise ConfigError(f"{path}.deadzone_rad_s: must be >= 0")
    if kind == TILTROTOR:
        kw["tilt_range"] = _field(doc, path, "tilt_range_rad", float)
        kw["tilt_axis"] = _vec(doc, path, "tilt_axis", 3, False, np.array([0.0, -1.0, 0.0]))
        kw["tilt_angle_default"] = _field(doc, path, "tilt_angle_default_rad", float, False, 0.0)
        if kw["tilt_range"] < 0:
            raise ConfigError(f"{path}.tilt_range_rad: must be >= 0")
        if abs(kw["tilt_angle_default"]) > kw["tilt_range"] + 1e-12:
            raise ConfigError(f"{path}.tilt_angle_default_rad: exceeds tilt_range_rad")
    return ActuatorSpec(**kw)


def parse_vehicle(doc, base_dir=None, name_hint=None) -> VehicleConfig:
    """Validate a schema_version-1 document (vehicles/__init__.py:262-324)."""
    if not isinstance(doc, dict):
        raise ConfigError("top level: expected a mapping")
    ver = _field(doc, "", "schema_version", int)
    if ver != SCHEMA_VERSION:
        raise ConfigError(f"schema_version: expected {SCHEMA_VERSION}, got {ver}")
    name = _field(doc, "", "name", str)
    if not name:
        raise ConfigError("name: must be non-empty")
    radius = _field(doc, "", "bounding_radius_m", float)
    if radius <= 0:
        raise ConfigError("bounding_radius_m: must be > 0")
    rd = _field(doc, "", "rigid_body", dict)
    try:
        rb = RigidBodyParams(mass=_field(rd, "rigid_body", "mass_kg", float),
                             inertia=_square(rd, "rigid_body", "inertia_kgm2", 3),
                             r_g=_vec(rd, "rigid_body", "center_of_gravity_m", 3),
                             r_b=_vec(rd, "rigid_body", "center_of_buoyancy_m", 3),
                             displaced_volume=_field(rd, "rigid_body", "displaced_volume_m3", float))
    except ParameterError as exc:
        raise ConfigError(f"rigid_body.{exc}") from exc
    hd = _field(doc, "", "hydrodynamics", dict)
    try:
        co = HydroCoeffs(M_A=_square(hd, "hydrodynamics", "added_mass", 6),
                         D_lin=_square(hd, "hydrodynamics", "linear_damping", 6),
                         D_quad=_square(hd, "hydrodynamics", "quadratic_damping", 6),
                         fluid_density=_field(hd, "hydrodynamics", "fluid_density_kgm3", float,
                                              False, 1000.0),
                         gravity=_field(hd, "hydrodynamics", "gravity_ms2", float, False, 9.81))
    except ParameterError as exc:
        raise ConfigError(f"hydrodynamics.{exc}") from exc
    docs = _field(doc, "", "actuators", list)
    if not docs:
        raise ConfigError("actuators: at least one actuator required")
    acts = []
    for i, ad in enumerate(docs):
        p = f"actuators[{i}]"
        if not isinstance(ad, dict):
            raise ConfigError(f"{p}: expected a mapping")
        try:
            acts.append(_parse_actuator(ad, p, base_dir))
        except ConfigError:
            raise
        except ValueError as exc:
            raise ConfigError(f"{p}: {exc}") from exc
    idx = sorted(a.index for a in acts)
    if len(set(idx)) != len(idx):
        raise ConfigError("actuators: duplicate actuator index")
    if idx != list(range(len(acts))):
        raise ConfigError("actuators: indices must be contiguous from 0")
    acts.sort(key=lambda a: a.index)
    return VehicleConfig(name=name, rb=rb, coeffs=co, actuators=acts, bounding_radius=radius,
                         schema_version=ver)


def vehicle_names() -> list:
    return list(BUILTIN_VEHICLES)


def load_vehicle(name_or_path) -> VehicleConfig:
    """Built-in vehicle by name (from ``fleet``), or a schema-v1 YAML document by path."""
    text = str(name_or_path)
    if text in BUILTIN_VEHICLES:
        return _from_fleet(text)
    path = Path(name_or_path)
    if not path.exists():
        raise ConfigError(f"vehicle '{text}': not a built-in {BUILTIN_VEHICLES} and no such file")
    import yaml

    try:
        doc = yaml.safe_load(path.read_text())
    except yaml.YAMLError as exc:
        raise ConfigError(f"{path}: invalid document ({exc})") from exc
    return parse_vehicle(doc, base_dir=path.parent)


# ---------------------------------------------------------------- overlays (host side)


def compose_with_payload(config: VehicleConfig, payload: Payload) -> RigidBodyParams:
    """Point-mass payload: conserved first moment + parallel axis (vehicles/__init__.py:418-440)."""
    rb = config.rb
    m, mp = rb.mass, payload.mass
    if mp == 0.0:
        return RigidBodyParams(mass=m, inertia=rb.inertia.copy(), r_g=rb.r_g.copy(),
                               r_b=rb.r_b.copy(), displaced_volume=rb.displaced_volume)
    total = m + mp
    cog = (m * rb.r_g + mp * payload.attach_position) / total

    def shift(mass, d):
        return mass * (float(d @ d) * np.eye(3) - np.outer(d, d))

    inertia = rb.inertia + shift(m, rb.r_g - cog) + shift(mp, payload.attach_position - cog)
    return RigidBodyParams(mass=total, inertia=inertia, r_g=cog, r_b=rb.r_b.copy(),
                           displaced_volume=rb.displaced_volume)


def validate_overlay(config: VehicleConfig, overlay: dict):
    for key in overlay:
        if key not in OVERLAY_KEYS:
            raise ConfigError(f"overlay: unknown key '{key}'")
    for key in RATIO_KEYS:
        if key in overlay and not overlay[key] > 0:
            raise ConfigError(f"overlay[{key}]: ratio must be > 0, got {overlay[key]}")
    if "cobm" in overlay and not overlay["cobm"] > 0:
        raise ConfigError(f"overlay[cobm]: scale must be > 0, got {overlay['cobm']}")
    if "payload_mass*" in overlay and overlay["payload_mass*"] < 0:
        raise ConfigError("overlay[payload_mass*]: ratio must be >= 0")
    jit = overlay.get("mount_position_jitter")
    if jit is not None and np.asarray(jit).shape not in ((3,), (config.action_dim, 3)):
        raise ConfigError("overlay[mount_position_jitter]: expected shape (3,) or (A, 3)")


def apply_overlay(config: VehicleConfig, overlay: dict) -> VehicleConfig:
    """New config with DR overlay values applied (vehicles/__init__.py:443-505)."""
    validate_overlay(config, overlay)
    g = overlay.get
    rb = config.rb
    r_b = rb.r_b.copy()
    if "cobm" in overlay:
        r_b[2] = rb.r_g[2] + overlay["cobm"] * (rb.r_b[2] - rb.r_g[2])
    new_rb = RigidBodyParams(mass=rb.mass * g("mass*", 1.0), inertia=rb.inertia * g("inertia*", 1.0),
                             r_g=rb.r_g.copy(), r_b=r_b,
                             displaced_volume=rb.displaced_volume * g("volume*", 1.0))
    co = config.coeffs
    new_co = HydroCoeffs(M_A=co.M_A * g("added_mass*", 1.0), D_lin=co.D_lin * g("damping*", 1.0),
                         D_quad=co.D_quad * g("damping*", 1.0), fluid_density=co.fluid_density,
                         gravity=co.gravity)
    jit = overlay.get("mount_position_jitter")
    jit = None if jit is None else np.asarray(jit, dtype=float)
    acts = []
    for i, a in enumerate(config.actuators):
        b = copy.deepcopy(a)
        b.time_constant = a.time_constant * g("time_constant*", 1.0)
        b.thrust_coeff = a.thrust_coeff * g("thrust_coeff*", 1.0)
        if jit is not None:
            b.mount_position = a.mount_position + (jit if jit.ndim == 1 else jit[i])
        acts.append(b)
    out = VehicleConfig(name=config.name, rb=new_rb, coeffs=new_co, actuators=acts,
                        bounding_radius=config.bounding_radius,
                        schema_version=config.schema_version)
    ratio = overlay.get("payload_mass*", 0.0)
    if ratio > 0.0:
        pos = np.asarray(overlay.get("payload_position", np.zeros(3)), dtype=float)
        out.rb = compose_with_payload(out, Payload(mass=ratio * out.rb.mass, attach_position=pos))
    return out


def tilt_rotation(axis, tilt_axis, angle):
    """Rodrigues rotation of a thrust axis about its tilt axis (actuation.py:176-184)."""
    axis = np.asarray(axis, dtype=float)
    k = np.asarray(tilt_axis, dtype=float)
    a = np.asarray(angle, dtype=float)[..., None]
    c, s = np.cos(a), np.sin(a)
    return axis * c + np.cross(k, axis) * s + k * (k * axis).sum(axis=-1)[..., None] * (1.0 - c)


def fin_basis(hinge):
    """Chord-forward / normal basis of a fin (engine.py:118-126)."""
    h = np.asarray(hinge, dtype=float)
    ref = np.array([1.0, 0.0, 0.0])
    xf = ref - float(ref @ h) * h
    if np.linalg.norm(xf) < 1e-9:
        ref = np.array([0.0, 0.0, 1.0])
        xf = ref - float(ref @ h) * h
    xf = xf / np.linalg.norm(xf)
    return xf, np.cross(h, xf)


def rb_mass_matrix(rb: RigidBodyParams) -> np.ndarray:
    """6x6 rigid-body mass matrix with CoG offset (hydrodynamics.py:88-101)."""
    x, y, z = rb.r_g
    S = np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])
    M = np.zeros((6, 6))
    M[:3, :3] = rb.mass * np.eye(3)
    M[:3, 3:] = -rb.mass * S
    M[3:, :3] = rb.mass * S
    M[3:, 3:] = rb.inertia - rb.mass * (S @ S)
    return M
