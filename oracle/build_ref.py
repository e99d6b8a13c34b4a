"""Recipe for oracle/_ref: install the UNMODIFIED reference package (moekit,
pure Python + NumPy) from /root/reference into oracle/_ref so bench.py's
reference arm and cpu_baseline can run it on the GPU box (where
/root/reference does not exist). Test/benchmark infrastructure only: nothing
in paper_2201_05596_b200/ imports it.

The source tree is read-only, so it is copied to a temporary directory first;
pip builds it offline (no index, no build isolation, no dependency
resolution - numpy is already in the image). oracle/_ref/ is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg"
OUT = os.path.join(HERE, "_ref")


def build_ref(force: bool = False) -> str | None:
    """-> OUT, or None when /root/reference is absent (e.g. on the GPU box,
    which uses the copy built here)."""
    if not os.path.isdir(REF_SRC):
        return OUT if os.path.isdir(os.path.join(OUT, "moekit")) else None
    if os.path.isdir(os.path.join(OUT, "moekit")) and not force:
        return OUT
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_SRC, src)
        if os.path.isdir(OUT):
            shutil.rmtree(OUT)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", OUT, src]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{res.stdout[-2000:]}{res.stderr[-2000:]}")
    return OUT


if __name__ == "__main__":
    print(build_ref(force="--force" in sys.argv))
