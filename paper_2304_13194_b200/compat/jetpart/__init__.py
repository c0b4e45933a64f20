"""`import jetpart` with this directory on sys.path gives the reference's
package with its hot path rebound to the GPU implementation
(paper_2304_13194_b200.jetpart_compat). Also makes `python -m jetpart.cli`
run the reference CLI on the GPU path."""
import os
import sys

_root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if _root not in sys.path:
    sys.path.insert(0, _root)

from paper_2304_13194_b200.jetpart_compat import install as _install  # noqa: E402

_install()
