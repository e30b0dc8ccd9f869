"""Drop-in shim: ``import sparsetc`` resolves to this package (paper_2405_16883_b200), so the
reference's own test suite can run unmodified against the B200 implementation
(tools/run_reference_tests.sh). Submodules map one to one; the reference's CLI is out of scope."""

import sys

import paper_2405_16883_b200 as _pkg
from paper_2405_16883_b200 import *  # noqa: F401,F403
from paper_2405_16883_b200 import (dense_eval, engine, expr, format_inference, formats, matrix_market,  # noqa: F401
                                   oracle, scheduler, tensor, tiling)

for _name in ("engine", "expr", "format_inference", "formats", "matrix_market", "oracle", "scheduler", "tensor",
              "tiling"):
    sys.modules[f"{__name__}.{_name}"] = getattr(_pkg, _name)
__version__ = _pkg.__version__

# The reference's CLI module (its test harness draws data with cli.synthetic_entries): loaded from
# the reference copy in baseline/_ref, its relative imports (.engine, .tensor, ...) bind to this
# package's modules above -- so the reference CLI itself runs on the B200 path.
import importlib.util as _ilu  # noqa: E402
from pathlib import Path as _Path  # noqa: E402

_cli = _Path(__file__).resolve().parents[3] / "baseline" / "_ref" / "sparsetc" / "cli.py"
if _cli.exists():
    _spec = _ilu.spec_from_file_location(f"{__name__}.cli", _cli)
    _mod = _ilu.module_from_spec(_spec)
    sys.modules[f"{__name__}.cli"] = _mod
    _spec.loader.exec_module(_mod)
    cli = _mod
