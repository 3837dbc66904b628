"""Exceptions shared by the host-side driver and the device core binding."""


class CoreOOM(Exception):
    """The logical memory budget (`budget_bytes`) would be exceeded by one more admission
    (reference `_kernels_py.py:28-29`, raised from `add_entry`, `_speedups.pyx:275-276`)."""


class CoreError(RuntimeError):
    """The device core reported a failure (CUDA error, device out of memory, bad arguments)."""


class BackendUnavailable(RuntimeError):
    """The CUDA shared library is missing or no B200 is visible.  There is deliberately no CPU
    fallback on the product path."""


class TimeoutExceeded(RuntimeError):
    pass
