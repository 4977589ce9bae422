"""Drop-in alias: ``import tilerun`` resolves to the B200 runtime.

Put ``compat/`` on PYTHONPATH (ahead of the reference) and code written for the
reference package -- including its own test suite -- runs on this package:
``tilerun.<name>`` and ``tilerun.<module>.<name>`` are the same objects as
``paper_1511_04348_b200.<...>``.
"""

import sys

import paper_1511_04348_b200 as _impl
from paper_1511_04348_b200 import *  # noqa: F401,F403

for _m in ("scheduler", "tiles", "coherence", "devices", "ann", "msqueue", "matio", "cli"):
    sys.modules[f"{__name__}.{_m}"] = getattr(_impl, _m)
    globals()[_m] = getattr(_impl, _m)

__all__ = list(_impl.__all__)
__version__ = _impl.__version__
