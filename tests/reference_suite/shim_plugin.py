"""pytest plugin (-p shim_plugin) for the frozen reference suite: puts the
reference package on sys.path and installs the B200 backend into it before
any test module is imported; at the end it records that the shim stayed
installed and which libsvb.so served the calls (SVB_REFSUITE_REPORT)."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


# at plugin import: before the reference conftest.py imports polysim
for _p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(_p, "polysim")):
        sys.path.insert(0, _p)
        break
sys.path.insert(0, ROOT)
from paper_2512_04216_b200 import polysim_shim  # noqa: E402

polysim_shim.install(pblock=True, sampling=True)


def pytest_sessionfinish(session, exitstatus):
    import polysim.pblock as ref_pb
    import polysim.sampling as ref_samp
    import polysim.statevector as ref_sv

    from paper_2512_04216_b200 import _lib, pblock, sampling
    from paper_2512_04216_b200 import statevector as sv

    rep = {
        "statevector_is_device": ref_sv.run is sv.run and ref_sv.apply_1q is sv.apply_1q,
        "pblock_is_device": ref_pb.run is pblock.run,
        "alias_table_is_device": ref_samp.AliasTable is sampling.AliasTable,
        "lib": _lib.LIB_PATH if _lib._lib is not None else None,
        "exitstatus": int(exitstatus),
        "collected": session.testscollected,
        "failed": session.testsfailed,
    }
    path = os.environ.get("SVB_REFSUITE_REPORT")
    if path:
        with open(path, "w") as fh:
            json.dump(rep, fh)
