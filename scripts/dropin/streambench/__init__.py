"""Package-swap shim: `import streambench` (and every `streambench.<module>`)
resolves to paper_2009_10917_b200, the B200 drop-in.

Put scripts/dropin on PYTHONPATH ahead of any real streambench; used by
scripts/run_reference_tests.sh to run the reference's own test suite against
the B200 package unchanged.
"""

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2009_10917_b200 as _pkg  # noqa: E402

_MODULES = ("cg", "cli", "core", "gs", "harness", "kernels", "mesh", "model", "parallel", "reference",
            "selftest")
for _name in _MODULES:
    _mod = importlib.import_module(f"paper_2009_10917_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_2009_10917_b200 import *  # noqa: E402,F401,F403

__all__ = list(_pkg.__all__)
__version__ = _pkg.__version__
