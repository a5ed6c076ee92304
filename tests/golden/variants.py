"""Non-builtin vehicles used by the golden fixtures.

Built from the constructor signatures that the reference classes and the
product's host classes share (``uuvsim.vehicles.VehicleConfig`` et al. and
``paper_2503_09203_b200.vehicles``), so the generator (reference) and the
tests (product/oracle) build bit-identical configs from one description.

* ``rotor_mix``  — bluerov with every rotor family: data-driven (t200 MLP)
  on thrusters 0-1, zero-order on 2, first-order elsewhere, and a reaction
  torque on thruster 4 (covers engine.py:340-351, 373-377).
* ``dense``      — bluerov with full (non-diagonal) SPD added-mass and damping
  matrices, a CoG offset and an inertia product term (covers the dense 6x6
  path of hydrodynamics.py:88-145).
* ``rotor_relu`` — ``rotor_mix`` with a relu rotor network (the relu branch of
  MLPWeights.forward, actuation.py:61-69).
"""

import numpy as np

T200 = dict(layer_sizes=[2, 8, 1], activation="tanh",
            weights=[[[1.5, -1.5], [3.0, -3.0], [0.8, -0.8], [2.2, -2.2],
                      [-1.5, 1.5], [-3.0, 3.0], [-0.8, 0.8], [-2.2, 2.2]],
                     [[0.8, 0.5, 1.0, 0.6, -0.8, -0.5, -1.0, -0.6]]],
            biases=[[0.0] * 8, [0.0]])


def _spd_perturb(diag, scale, seed):
    rng = np.random.default_rng(seed)
    n = len(diag)
    A = rng.uniform(-1.0, 1.0, size=(n, n)) * scale
    S = 0.5 * (A + A.T)
    M = np.diag(diag) + S * np.sqrt(np.outer(diag, diag))
    # keep it well inside the SPD cone
    return M + np.diag(np.asarray(diag) * 0.5)


def build(name, mod_vehicles, mod_actuation, mod_hydro, base):
    """Return the variant ``name`` built on top of ``base`` (a bluerov config)."""
    import copy

    V = mod_vehicles
    acts = []
    for a in base.actuators:
        acts.append(copy.deepcopy(a))
    rb, co = base.rb, base.coeffs
    if name in ("rotor_mix", "rotor_relu"):
        # rotor_relu: the same mix with a relu rotor network (actuation.py:61-69 relu branch)
        act_fn = "relu" if name == "rotor_relu" else "tanh"
        net = mod_actuation.MLPWeights(layer_sizes=T200["layer_sizes"], weights=T200["weights"],
                                       biases=T200["biases"], activation=act_fn)
        for j in (0, 1):
            acts[j].rotor_model = "data_driven"
            acts[j].mlp = net
            acts[j].weights_ref = "t200_mlp.yaml"
        acts[2].rotor_model = "zero_order"
        acts[4].reaction_coeff = 3.0e-6
        return V.VehicleConfig(name=name, rb=copy.deepcopy(rb), coeffs=copy.deepcopy(co),
                               actuators=acts, bounding_radius=base.bounding_radius)
    if name == "dense":
        M_A = _spd_perturb(np.diag(co.M_A), 0.2, 1)
        D_lin = _spd_perturb(np.diag(co.D_lin), 0.2, 2)
        D_quad = _spd_perturb(np.diag(co.D_quad), 0.2, 3)
        inertia = np.array([[0.16, 0.004, -0.002], [0.004, 0.17, 0.003], [-0.002, 0.003, 0.15]])
        new_rb = mod_hydro.RigidBodyParams(mass=rb.mass, inertia=inertia,
                                           r_g=np.array([0.01, -0.005, 0.02]),
                                           r_b=np.array([0.0, 0.002, -0.02]),
                                           displaced_volume=rb.displaced_volume * 1.01)
        new_co = mod_hydro.HydroCoeffs(M_A=M_A, D_lin=D_lin, D_quad=D_quad)
        return V.VehicleConfig(name="dense", rb=new_rb, coeffs=new_co, actuators=acts,
                               bounding_radius=base.bounding_radius)
    raise KeyError(name)


VARIANTS = ("rotor_mix", "dense", "rotor_relu")
