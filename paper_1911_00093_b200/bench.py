"""`hmx.bench` under the reference's module name (reference
pkg/src/hmx/bench.py): callers that import `hmx.bench.run_matvec_bench` etc.
find the GPU drivers of benchrec.py here."""

from .benchrec import *  # noqa: F401,F403
from .benchrec import __all__  # noqa: F401
