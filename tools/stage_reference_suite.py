"""Stage the reference's own test suite for a run against the GPU package.

Copies /root/reference/pkg/tests/*.py (build container only) into
.reftests/ -- git-ignored, so the reference's tests are never committed, but
not gpurun-ignored, so they travel to the GPU box -- and writes a conftest
that aliases `sboxeval` and its submodules to paper_1912_03732_b200, so the
reference's imports (`from sboxeval import ...`, `import sboxeval.bench as
bench`, `from sboxeval.cli import main`, `from sboxeval.memory import
MemoryBudgetError`) resolve to the GPU implementation.

    python tools/stage_reference_suite.py
    gpurun -- 'python -m pytest .reftests -q -p no:cacheprovider'
"""
import glob
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, ".reftests")
CONFTEST = '''import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1912_03732_b200 as _pkg  # noqa: E402

sys.modules["sboxeval"] = _pkg
for _sub in ("walsh", "parallel", "nonlinearity", "memory", "bench", "sbox", "cli"):
    sys.modules["sboxeval." + _sub] = importlib.import_module("paper_1912_03732_b200." + _sub)
'''


def main():
    os.makedirs(DST, exist_ok=True)
    for f in glob.glob("/root/reference/pkg/tests/*.py"):
        shutil.copy(f, DST)
    with open(os.path.join(DST, "conftest.py"), "w") as fh:
        fh.write(CONFTEST)
    print(sorted(os.listdir(DST)))


if __name__ == "__main__":
    main()
