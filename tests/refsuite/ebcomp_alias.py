"""pytest plugin: make ``import ebcomp`` resolve to this package.

Used to run the reference's own test suite against the drop-in:

    python -m pytest -p ebcomp_alias <staged reference tests> \
        --ignore=.../test_cli.py

with tests/refsuite on PYTHONPATH.  The staged copy lives in the git-ignored
baseline/_ref/ref_tests (written by __graft_entry__.build() when the reference
checkout is present); nothing of it is committed.
"""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.append(ROOT)

import paper_2312_05492_b200 as _P  # noqa: E402

sys.modules["ebcomp"] = _P
for _sub in ("errors", "grid", "predictor", "tuning", "huffman", "pass2", "archive", "pipeline",
             "lorenzo", "metrics"):
    sys.modules["ebcomp." + _sub] = importlib.import_module("paper_2312_05492_b200." + _sub)
