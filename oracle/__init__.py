"""CPU oracle for the GCG hot path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg.  `gcg_oracle` is a numpy restatement of the reference (pinned by
tests/test_oracle_pin.py); `load_reference()` returns the unmodified reference
package built into oracle/_ref by oracle/build_ref.sh, when present.
"""

import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")


def load_reference():
    """Return the reference `gcgeig` module from oracle/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "gcgeig")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import gcgeig  # noqa: E402

    return gcgeig
