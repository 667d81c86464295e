"""B200-native HPG-MxP solve path (drop-in for the reference package ``mxpbench``).

Same public API as the reference (ref: __init__.py:12-15): ``BenchConfig``,
``main``, ``run_benchmark``, ``run_validation``.  Every numeric step runs in
hand-written sm_100a kernels in ``libhpgmxp.so`` (include/hpgmxp.h); there
is no CPU path.
"""

__version__ = "0.1.0"

from .bench import BenchConfig, main, run_benchmark, run_validation  # noqa: E402

__all__ = ["BenchConfig", "main", "run_benchmark", "run_validation", "__version__"]
