"""pytest plugin: run the REFERENCE's own unit tests on the unmodified
reference package (baseline/_ref) with its hot path dispatched to
libsketchqr_b200.so through integration/sketchqr_b200_binding.py (ctypes only;
paper_2405_10923_b200's Python is not imported).  scripts/ref_suite/run.sh
patched."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, os.path.join(ROOT, "integration"))

import sketchqr  # noqa: E402
import sketchqr_b200_binding as b200  # noqa: E402

b200.install(sketchqr, os.path.join(ROOT, "paper_2405_10923_b200", "libsketchqr_b200.so"))
assert "paper_2405_10923_b200" not in sys.modules
