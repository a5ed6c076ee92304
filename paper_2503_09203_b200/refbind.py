"""Reference-side binding: the unmodified reference's ``step_batch`` on the B200 kernel.

This is the stub INTEGRATION.md §2 describes, as a module a maintainer of the
reference (``uuvsim``) would vendor: it keeps the reference's numpy
``BatchState`` (engine.py:269-295) as the source of truth and runs each control
step through the C ABI with DLPack tensors (``uuv_state_from_dlpack`` +
``uuv_step_dl``, via this package's engine), float64 for parity:

    from uuvsim import engine
    from paper_2503_09203_b200 import refbind
    refbind.install(engine)             # engine.step_batch dispatches bound batches
    state = engine.make_batch(vehicle, sim)
    engine.reset_envs(state, mask, sampler)
    refbind.bind(state)                 # attach the device mirror
    engine.step_batch(state, commands)  # p, q, nu, act, steps, diverged updated in place

Per-env parameters are carried as the reference's overlay dicts
(``state.overlays``, engine.py:507): whenever the episode counters change the
rows are re-uploaded through the host reset path, which applies them with the
reference's overlay semantics (vehicles/__init__.py:418-505).
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine as E


class B200Step:
    """Device mirror of one reference ``BatchState`` (float64)."""

    def __init__(self, state, device=None):
        sim = state.sim
        self.n = int(sim.batch_size)
        self.bs = E.make_batch(state.vehicle, E.SimConfig(dt=sim.dt, substeps=sim.substeps,
                                                          batch_size=self.n),
                               master_seed=int(state.master_seed), device=device,
                               dtype=torch.float64)
        self._episodes = None

    def _sync_params(self, state):
        """Upload every row's overlay (the reference's per-env BatchParams rows)."""
        ovs = state.overlays

        def sampler(i, ep, rng):
            return E.EnvInit(pose=E.Pose(), overlay=dict(ovs[i]))

        E.reset_envs(self.bs, np.ones(self.n, bool), sampler)
        self._episodes = np.array(state.episodes, copy=True)

    def step(self, state, commands, error=ValueError):
        """One control step of the reference batch (engine.py:465-484), in place."""
        commands = np.asarray(commands, dtype=float)
        a = state.layout.action_dim
        if commands.shape != (self.n, a):
            raise error(f"commands: expected shape {(self.n, a)}, got {commands.shape}")
        if self._episodes is None or not np.array_equal(self._episodes, state.episodes):
            self._sync_params(state)
        bs, dev = self.bs, self.bs.device

        def up(x):
            return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

        bs.p[:] = up(state.p)
        bs.q[:] = up(state.q)
        bs.nu[:] = up(state.nu)
        bs.act[:] = up(state.act)
        if np.any(state.current_ned != 0.0) or bs._cur is not None:
            bs.current_ned[:] = up(state.current_ned)
        bs.steps[:] = up(state.steps.astype(np.int32))
        bs.diverged[:] = up(state.diverged)
        E.step_batch(bs, up(commands))
        state.p[:] = bs.p.cpu().numpy()
        state.q[:] = bs.q.cpu().numpy()
        state.nu[:] = bs.nu.cpu().numpy()
        state.act[:] = bs.act.cpu().numpy()
        state.diverged[:] = bs.diverged.cpu().numpy()
        state.steps[:] = bs.steps.cpu().numpy()
        return state


def bind(state, device=None) -> B200Step:
    """Attach a device mirror to a reference BatchState (``state._b200``)."""
    state._b200 = B200Step(state, device)
    return state._b200


def install(ref_engine):
    """Make ``ref_engine.step_batch`` dispatch bound batches to the kernel (the two-line
    change INTEGRATION.md §2 shows in engine.py:471-474); returns the original."""
    original = ref_engine.step_batch

    def step_batch(state, commands):
        b = getattr(state, "_b200", None)
        if b is None:
            return original(state, commands)
        return b.step(state, commands, ref_engine.EngineError)

    step_batch.__wrapped__ = original
    ref_engine.step_batch = step_batch
    return original
