"""Run the reference's OWN test modules against this package (SURVEY.md 8(c) "Strategy").

    python scripts/run_reference_suite.py SUITE [pytest args...]

SUITE is a directory or a .tar.gz holding the reference's pkg/tests files (conftest.py,
test_sampling.py, test_storage.py, test_cache.py, test_features.py, ...).  /root/reference does
not exist on the GPU box, so the build container packs them and the gpurun command line carries
them (scripts/reference_suite_gpurun.sh); nothing of the reference is stored in this repo.

The modules run unmodified: a pytest plugin aliases ``ctdg`` and its submodules to
``paper_2311_17410_b200`` (every graph, cache and table the tests build lives on cuda:0 and every
sample runs through libgfb200), so each ``from ctdg import ...`` binds the B200 implementation.
Deviations documented in DESIGN.md section 2 are reported, not hidden: the summary lists every
failure with its reason.
"""

from __future__ import annotations

import os
import shutil
import sys
import tarfile
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHIM = '''
import sys
sys.path.insert(0, {root!r})
import paper_2311_17410_b200 as _gf
from paper_2311_17410_b200 import storage, sampling, cache, features, synth, metrics, partition, cluster, harness, wire, cli
sys.modules["ctdg"] = _gf
for _name, _mod in (("storage", storage), ("sampling", sampling), ("cache", cache), ("features", features),
                    ("synth", synth), ("metrics", metrics), ("partition", partition), ("cluster", cluster),
                    ("harness", harness), ("wire", wire), ("cli", cli)):
    sys.modules["ctdg." + _name] = _mod
'''


def main() -> int:
    if len(sys.argv) < 2:
        print(__doc__)
        return 2
    src = sys.argv[1]
    work = tempfile.mkdtemp(prefix="ref_suite_")
    if os.path.isdir(src):
        for f in os.listdir(src):
            if f.endswith(".py"):
                shutil.copy(os.path.join(src, f), work)
    else:
        with tarfile.open(src) as tf:
            tf.extractall(work, filter="data")
    with open(os.path.join(work, "ctdg_shim.py"), "w") as fh:
        fh.write(SHIM.format(root=ROOT))
    import pytest

    args = ["-p", "ctdg_shim", "-p", "no:cacheprovider", "-q", "-rfEx", "--rootdir", work, work] + sys.argv[2:]
    sys.path.insert(0, work)
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    return pytest.main(args)


if __name__ == "__main__":
    sys.exit(main())
