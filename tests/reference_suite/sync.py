"""Copy the reference's own strategy and acceptance tests next to this file
(tests/reference_suite/vendor/, git-ignored) so they run unmodified against
this package on the GPU box (conftest.py here aliases ``idwlayout`` to
``paper_1402_4986_b200``).

Runs here, where /root/reference exists (``__graft_entry__.build()`` calls
it); the copies travel to the GPU box with the working tree like the built
.so files, and never enter git history.  The only edit is mechanical: the
reference's tests import helpers ``from conftest import ...``; the reference
conftest.py is copied as ``ref_conftest.py`` and those imports renamed, so
it cannot collide with this repo's own tests/conftest.py.

Copied: test_strategies.py, test_acceptance.py (reference SURVEY §4: the
strategy contract and the eight acceptance criteria), and the helpers they
import (conftest.py, oracle_idw.py, oracle_txn.py).
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parent / "vendor"
FILES = ("test_strategies.py", "test_acceptance.py", "oracle_idw.py", "oracle_txn.py")


def sync() -> bool:
    if not SRC.is_dir():
        return False
    DST.mkdir(exist_ok=True)
    for name in FILES:
        text = (SRC / name).read_text()
        (DST / name).write_text(text.replace("from conftest import", "from ref_conftest import"))
    shutil.copyfile(SRC / "conftest.py", DST / "ref_conftest.py")
    return True


if __name__ == "__main__":
    ok = sync()
    print(f"reference tests {'copied to ' + str(DST) if ok else 'not found (no /root/reference here)'}")
    sys.exit(0)
