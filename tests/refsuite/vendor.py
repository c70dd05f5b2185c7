"""Copy the reference's own test suite (/root/reference/pkg/tests) into
tests/refsuite/_vendored/ so it runs against this package (SURVEY §4 reuse
plan, VERDICT r1 "next" item 2).

The copied files are the reference's code, so they are NOT committed
(`_vendored/` is git-ignored); they travel to the GPU box with the working
tree like the built .so files.  `tests/refsuite/conftest.py` aliases the
`specdraft` package to `paper_2411_05894_b200` (tests/refsuite/shim) and marks
every vendored test `gpu`: the package has no CPU fallback.

    python tests/refsuite/vendor.py            # needs /root/reference (this container)
"""

from __future__ import annotations

import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_vendored")


def main() -> int:
    if not os.path.isdir(SRC):
        print(f"{SRC} not found: nothing to vendor", file=sys.stderr)
        return 1
    os.makedirs(DST, exist_ok=True)
    n = 0
    for name in sorted(os.listdir(SRC)):
        if name.endswith(".py"):
            shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
            n += 1
    print(f"vendored {n} files into {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
