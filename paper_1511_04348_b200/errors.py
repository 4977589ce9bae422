"""Exception classes with the reference's hierarchy.

``ConfigError(ValueError)`` mirrors devices.py:26-27 and
``CapacityError(RuntimeError)`` mirrors coherence.py:33-34.
"""


class ConfigError(ValueError):
    """Invalid device / machine configuration (devices.py:26-27)."""


class CapacityError(RuntimeError):
    """A device cannot hold a task's working set (coherence.py:33-34)."""


class NoDeviceError(RuntimeError):
    """The product path needs a CUDA device and none is available.

    There is deliberately no CPU fallback: the arithmetic of this framework is
    the sm_100a tile kernel.
    """
