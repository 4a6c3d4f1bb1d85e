"""CPU float64 oracle for the orthogonal-convolution hot path (TEST INFRASTRUCTURE).

This package is test infrastructure, not product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with the CUDA path
(``paper_2601_13776_b200/``) and imports nothing from it.

See ``oracle/orth_oracle.py`` for the functions and the passages they follow.
"""
from .orth_oracle import *  # noqa: F401,F403
from .orth_oracle import __all__  # noqa: F401
