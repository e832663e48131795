"""pytest plugin: run the reference's own test files against the B200 path.

    PYTHONPATH=oracle/_ref:. python -m pytest oracle/_ref/tests/test_solver.py \
        -p paper_2111_06552_b200.refdrop_plugin

Loaded before collection, it rebinds gcgeig.gcg_solve and the orth entry points
to the device implementations (refdrop.install), so the reference's test modules
import the B200 versions (`from gcgeig import gcg_solve`).  Unit tests of the
reference's private helpers (_build_p, select_shift) still test the reference.
"""

import gcgeig as _gcgeig

from paper_2111_06552_b200 import refdrop as _rd

_rd.install(_gcgeig)
