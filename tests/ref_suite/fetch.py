"""Copy the reference's own test files next to the shim (build container only).

    python tests/ref_suite/fetch.py

The copies land in tests/ref_suite/_ref/, which is git-ignored (reference sources are never
committed) but not gpurun-ignored, so they travel to the GPU box with the snapshot like the
built libmdd.so does.  tests/test_reference_suite.py runs them there against the drop-in
package (maxwelldd -> paper_1711_03789_b200 through tests/ref_suite/shim)."""
import os
import shutil

SRC = "/root/reference/pkg/tests"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")

if __name__ == "__main__":
    os.makedirs(DST, exist_ok=True)
    n = 0
    for f in sorted(os.listdir(SRC)):
        if f.endswith(".py"):
            shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))
            n += 1
    print(f"copied {n} files to {DST}")
