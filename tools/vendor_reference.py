"""Vendor the unmodified reference package into baseline/_ref (git-ignored;
gpurun ships it to the GPU box with the snapshot).

    python tools/vendor_reference.py [--force]

* ``baseline/_ref/hetserve``: ``pip install --no-index --no-build-isolation
  --no-deps --target baseline/_ref`` of /root/reference/pkg (built from a copy
  under /tmp because /root/reference is read-only; numpy / pyyaml are already
  in the image, so only dependency resolution is skipped);
* ``baseline/_ref/tests``: the reference's own test-suite
  (/root/reference/pkg/tests), run against the engine by
  tests/test_reference_suite.py through paper_2504_15303_b200.refbind.
"""

from __future__ import annotations

import pathlib
import shutil
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF = pathlib.Path("/root/reference/pkg")
DEST = ROOT / "baseline" / "_ref"


def vendor(force: bool = False) -> bool:
    if (DEST / "hetserve" / "__init__.py").exists() and (DEST / "tests" / "conftest.py").exists() and not force:
        return True
    if not REF.exists():
        return False
    with tempfile.TemporaryDirectory() as tmp:
        src = pathlib.Path(tmp) / "pkg"
        shutil.copytree(REF, src)
        if DEST.exists():
            shutil.rmtree(DEST)
        subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation",
                        "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(DEST), str(src)], check=True)
    shutil.copytree(REF / "tests", DEST / "tests")
    return True


if __name__ == "__main__":
    print("vendored" if vendor(force="--force" in sys.argv) else "reference not present")
