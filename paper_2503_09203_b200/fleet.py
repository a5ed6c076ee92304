"""Built-in UUV fleet as plain numeric tables.

The five vehicles and two rotor networks the reference ships as YAML
documents (``uuvsim/vehicles/data/*.yaml``, listed at
``uuvsim/vehicles/__init__.py:44``) are restated here as Python literals so the
package carries no file I/O on its import path and travels to the GPU box
as source.  ``tests/test_fleet_data.py`` checks every number against the
reference documents when ``/root/reference`` is mounted, and the golden
trajectories under ``tests/golden/`` pin them again through the physics.

Conventions: body frame x forward, y starboard, z down; SI units.  Each
actuator row is a dict in the field names of the reference schema
(``vehicles/__init__.py:185-259``) minus the unit suffixes.
"""

from __future__ import annotations

_H = 0.7071067811865476  # cos(45 deg) as written in the reference documents
_HALF_PI = 1.5707963267948966


def _prop(mount, axis, tau, c_t, dz, n_max):
    return dict(kind="propeller", mount=mount, axis=axis, model="first_order",
                time_constant=tau, thrust_coeff=c_t, deadzone=dz, max_speed=n_max)


def _fin(mount, hinge, tau, area, cla, cd0, kd, stall, max_angle):
    return dict(kind="rudder", mount=mount, axis=hinge, model="first_order",
                time_constant=tau,
                rudder=dict(area=area, c_l_alpha=cla, c_d0=cd0, k_d=kd,
                            stall_angle=stall, max_angle=max_angle, fluid_density=1000.0))


def _tilt(mount, axis, tilt_axis, tilt0):
    return dict(kind="tiltrotor", mount=mount, axis=axis, model="first_order",
                time_constant=0.12, thrust_coeff=1.5e-4, deadzone=20.0, max_speed=350.0,
                tilt_range=_HALF_PI, tilt_axis=tilt_axis, tilt_default=tilt0)


def _vectored_quad(x, y, tau=0.15, c_t=2.5e-4, dz=25.0, n_max=400.0):
    """Four horizontal thrusters at +-45 deg (the BlueROV2 frame)."""
    return [
        _prop([x, y, 0.0], [_H, -_H, 0.0], tau, c_t, dz, n_max),
        _prop([x, -y, 0.0], [_H, _H, 0.0], tau, c_t, dz, n_max),
        _prop([-x, y, 0.0], [-_H, -_H, 0.0], tau, c_t, dz, n_max),
        _prop([-x, -y, 0.0], [-_H, _H, 0.0], tau, c_t, dz, n_max),
    ]


def _vertical(points, tau=0.15, c_t=2.5e-4, dz=25.0, n_max=400.0):
    return [_prop(list(p), [0.0, 0.0, -1.0], tau, c_t, dz, n_max) for p in points]


def _cruciform(x, off, tau, area, cla, kd):
    """Top/bottom rudders (hinge z) then starboard/port elevators (hinge y)."""
    return [
        _fin([x, 0.0, -off], [0.0, 0.0, 1.0], tau, area, cla, 0.02, kd, 0.52, 0.35),
        _fin([x, 0.0, off], [0.0, 0.0, 1.0], tau, area, cla, 0.02, kd, 0.52, 0.35),
        _fin([x, off, 0.0], [0.0, 1.0, 0.0], tau, area, cla, 0.02, kd, 0.52, 0.35),
        _fin([x, -off, 0.0], [0.0, 1.0, 0.0], tau, area, cla, 0.02, kd, 0.52, 0.35),
    ]


def _hull(mass, volume, r_g, r_b, inertia_diag, added, d_lin, d_quad):
    return dict(mass=mass, volume=volume, r_g=r_g, r_b=r_b, inertia_diag=inertia_diag,
                added_mass_diag=added, linear_damping_diag=d_lin,
                quadratic_damping_diag=d_quad, fluid_density=1000.0, gravity=9.81)


FLEET = {
    # bluerov.yaml: 4 vectored + 2 vertical
    "bluerov": dict(
        bounding_radius=0.35,
        hull=_hull(11.5, 0.0115, [0.0, 0.0, 0.0], [0.0, 0.0, -0.02], [0.16, 0.16, 0.16],
                   [5.5, 12.7, 14.57, 0.12, 0.12, 0.12],
                   [4.03, 6.22, 5.18, 0.07, 0.07, 0.07],
                   [18.18, 21.66, 36.99, 1.55, 1.55, 1.55]),
        actuators=_vectored_quad(0.156, 0.111)
        + _vertical([(0.0, 0.111, -0.085), (0.0, -0.111, -0.085)]),
    ),
    # bluerov_heavy.yaml: 4 vectored + 4 vertical
    "bluerov_heavy": dict(
        bounding_radius=0.4,
        hull=_hull(13.5, 0.0135, [0.0, 0.0, 0.0], [0.0, 0.0, -0.025], [0.26, 0.23, 0.37],
                   [6.36, 7.12, 18.68, 0.189, 0.135, 0.222],
                   [13.7, 0.0, 33.0, 0.0, 0.8, 0.0],
                   [141.0, 217.0, 190.0, 1.19, 0.47, 1.5]),
        actuators=_vectored_quad(0.156, 0.111)
        + _vertical([(0.12, 0.218, -0.085), (0.12, -0.218, -0.085),
                     (-0.12, 0.218, -0.085), (-0.12, -0.218, -0.085)]),
    ),
    # lauv.yaml: stern thruster + cruciform fins
    "lauv": dict(
        bounding_radius=0.6,
        hull=_hull(18.0, 0.018, [0.0, 0.0, 0.0], [0.0, 0.0, -0.01], [0.04, 1.6, 1.6],
                   [1.0, 16.0, 16.0, 0.01, 1.2, 1.2],
                   [2.4, 23.0, 23.0, 0.3, 3.1, 3.1],
                   [2.4, 80.0, 80.0, 0.01, 9.1, 9.1]),
        actuators=[_prop([-0.55, 0.0, 0.0], [1.0, 0.0, 0.0], 0.2, 1.0e-4, 10.0, 280.0)]
        + _cruciform(-0.45, 0.075, 0.1, 0.008, 3.0, 1.2),
    ),
    # iauv.yaml: heavier torpedo hull, same actuator topology as lauv
    "iauv": dict(
        bounding_radius=0.7,
        hull=_hull(30.0, 0.03, [0.0, 0.0, 0.02], [0.0, 0.0, -0.015], [0.8, 3.5, 3.4],
                   [4.0, 30.0, 35.0, 0.2, 3.0, 2.8],
                   [5.0, 30.0, 34.0, 0.8, 4.5, 4.2],
                   [9.0, 110.0, 120.0, 0.5, 12.0, 11.0]),
        actuators=[_prop([-0.6, 0.0, 0.0], [1.0, 0.0, 0.0], 0.2, 1.8e-4, 10.0, 300.0)]
        + _cruciform(-0.5, 0.09, 0.1, 0.012, 3.2, 1.2),
    ),
    # hauv.yaml: eight tiltrotors, four corners level, four vectored at 90 deg tilt
    "hauv": dict(
        bounding_radius=0.5,
        hull=_hull(25.0, 0.025, [0.0, 0.0, 0.01], [0.0, 0.0, -0.03], [0.9, 1.1, 1.6],
                   [8.0, 12.0, 20.0, 0.3, 0.8, 1.0],
                   [12.0, 15.0, 25.0, 0.6, 0.9, 1.2],
                   [60.0, 80.0, 120.0, 1.0, 2.0, 3.0]),
        actuators=[
            _tilt([0.3, 0.22, 0.0], [_H, -_H, 0.0], [-_H, -_H, 0.0], 0.0),
            _tilt([0.3, -0.22, 0.0], [_H, _H, 0.0], [_H, -_H, 0.0], 0.0),
            _tilt([-0.3, 0.22, 0.0], [-_H, -_H, 0.0], [-_H, _H, 0.0], 0.0),
            _tilt([-0.3, -0.22, 0.0], [-_H, _H, 0.0], [_H, _H, 0.0], 0.0),
        ] + [
            _tilt([sx * 0.22, sy * 0.3, 0.0], [1.0, 0.0, 0.0], [0.0, -1.0, 0.0], _HALF_PI)
            for sx, sy in ((1, 1), (1, -1), (-1, 1), (-1, -1))
        ],
    ),
}

BUILTIN_VEHICLES = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv")


def _antisym_net(w_in, w_out):
    """2-H-1 tanh net whose hidden units come in +/- pairs (t200/m2820 placeholders)."""
    first = [[w, -w] for w in w_in] + [[-w, w] for w in w_in]
    second = [list(w_out) + [-w for w in w_out]]
    h = len(first)
    return dict(layer_sizes=[2, h, 1], activation="tanh", weights=[first, second],
                biases=[[0.0] * h, [0.0]])


# t200_mlp.yaml / m2820_mlp.yaml (placeholder rotor-response networks)
ROTOR_NETS = {
    "t200_mlp": _antisym_net([1.5, 3.0, 0.8, 2.2], [0.8, 0.5, 1.0, 0.6]),
    "m2820_mlp": _antisym_net([1.8, 3.6, 1.0, 2.6], [0.85, 0.55, 1.05, 0.65]),
}
