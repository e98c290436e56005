"""Freeze the reference's own test files for the dense state-vector path into
tests/reference_suite/_frozen/ (git-ignored: they are the reference's source,
not this repo's; the directory travels to the GPU box with the working tree).

    python tests/reference_suite/freeze.py [/root/reference/pkg/tests]

The frozen files are run unmodified by tests/test_gpu_reference_suite.py in a
separate pytest process with shim_plugin.py loaded, which installs this
package into the reference (`polysim_shim.install(pblock=True, sampling=True)`)
before collection, so `polysim.statevector`, `polysim.pblock` and
`polysim.sampling.AliasTable` resolve to the B200 backend.  Called by
__graft_entry__.build() whenever the reference tree is present."""
from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
FROZEN = os.path.join(HERE, "_frozen")
FILES = ("conftest.py", "test_statevector.py", "test_sampling.py", "test_pblock.py")


def freeze(src: str = "/root/reference/pkg/tests") -> bool:
    if not all(os.path.isfile(os.path.join(src, f)) for f in FILES):
        return False
    os.makedirs(FROZEN, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(src, f), os.path.join(FROZEN, f))
    with open(os.path.join(FROZEN, "SOURCE"), "w") as fh:
        fh.write(f"frozen from {src}: {', '.join(FILES)}\n")
    return True


if __name__ == "__main__":
    ok = freeze(*sys.argv[1:2])
    print("frozen" if ok else "reference tests not found")
    sys.exit(0 if ok else 1)
