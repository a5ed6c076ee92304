"""Built-in fleet data equals the reference documents (build container only)."""

import os

import numpy as np
import pytest

from paper_2503_09203_b200 import vehicles as pv

REF_DATA = "/root/reference/pkg/src/uuvsim/vehicles/data"


@pytest.mark.skipif(not os.path.isdir(REF_DATA), reason="reference not mounted")
@pytest.mark.parametrize("name", pv.BUILTIN_VEHICLES)
def test_fleet_matches_reference_yaml(name):
    ours = pv.load_vehicle(name)
    theirs = pv.load_vehicle(os.path.join(REF_DATA, f"{name}.yaml"))
    assert ours.name == theirs.name and ours.bounding_radius == theirs.bounding_radius
    for k in ("mass", "displaced_volume", "inertia", "r_g", "r_b"):
        assert np.array_equal(getattr(ours.rb, k), getattr(theirs.rb, k)), k
    for k in ("M_A", "D_lin", "D_quad", "fluid_density", "gravity"):
        assert np.array_equal(getattr(ours.coeffs, k), getattr(theirs.coeffs, k)), k
    assert len(ours.actuators) == len(theirs.actuators)
    for a, b in zip(ours.actuators, theirs.actuators):
        for k in ("index", "kind", "mount_position", "mount_axis", "rotor_model", "time_constant",
                  "thrust_coeff", "deadzone", "max_speed", "reaction_coeff", "tilt_range",
                  "tilt_axis", "tilt_angle_default"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (name, a.index, k)
        assert a.rudder == b.rudder


@pytest.mark.skipif(not os.path.isdir(REF_DATA), reason="reference not mounted")
@pytest.mark.parametrize("name", ["t200_mlp", "m2820_mlp"])
def test_rotor_nets_match_reference_yaml(name):
    ours = pv.builtin_rotor_net(name)
    theirs = pv.load_mlp_weights(os.path.join(REF_DATA, f"{name}.yaml"))
    assert ours.layer_sizes == theirs.layer_sizes and ours.activation == theirs.activation
    for a, b in zip(ours.weights + ours.biases, theirs.weights + theirs.biases):
        assert np.array_equal(a, b)


def test_load_vehicle_errors():
    with pytest.raises(pv.ConfigError):
        pv.load_vehicle("no_such_vehicle")
