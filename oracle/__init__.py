"""Oracle package — TEST INFRASTRUCTURE ONLY.

Two checkers for the B200 boundary-message path:

* ``port``  — ``qgnn_oracle.c``, a plain-C restatement of the reference
  algorithm (rng.hpp, quant.hpp, codec.hpp, aggregate.hpp, model.hpp,
  matrix.hpp, coeffs.hpp), built to ``oracle/_build/libqgnn_oracle.so``.
* ``ref``   — the UNMODIFIED reference headers compiled through
  ``ref_shim.cpp`` into ``oracle/_ref/libqgnn_ref.so`` (recipe:
  ``oracle/Makefile``).  It pins the port and generates ``tests/golden``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package; the product (``paper_2306_01381_b200``) never
does.
"""
from .oracle import RefError, build, port, ref, ref_available  # noqa: F401
