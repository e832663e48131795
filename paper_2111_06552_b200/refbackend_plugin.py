"""pytest plugin: register the `sm100` backend into the reference before collection.

    PYTHONPATH=oracle/_ref python -m pytest oracle/_ref/tests/test_multivec.py \
        -p paper_2111_06552_b200.refbackend_plugin

The reference's `backend` fixture (conftest.py:7-13) parametrises over
`kernels.available_backends()` when its conftest is imported, so registration
happens at plugin import (before conftest loading); every reference test that
takes the fixture then also runs with the B200 kernels.
"""

import gcgeig._kernels as _K

from paper_2111_06552_b200 import refbackend as _rb

_rb.register(_K)
