"""B200-native batched 6-DOF Fossen step for MarineGym-style UUV environments.

Drop-in for the reference ``uuvsim`` hot path (``engine.step_batch``,
``engine.reset_envs``, ``tasks.make_env``): the same Python API over torch
CUDA tensors, backed by hand-written sm_100a kernels behind a C ABI
(``include/uuv_b200.h``, ``libuuvb200.so``).
"""

__version__ = "0.1.0"
