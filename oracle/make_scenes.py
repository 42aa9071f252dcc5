#!/usr/bin/env python3
"""Build the committed workload scenes (TEST/BENCH INFRASTRUCTURE).

data/c2.sdfs: scenegen.c2_scene() clustered by the REFERENCE's buildClusters
(scene.hpp:110-178; maxPerCluster 8, mergeRadius 10 = RenderConfig defaults)
through oracle/_ref/ref_parity `recluster`, so the CPU reference and the GPU see
the very clusters the reference would build. Takes ~10 s (O(N^3) builder).
"""
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2007_14394_b200 import scene_io, scenegen  # noqa: E402


def main():
    out = os.path.join(ROOT, "paper_2007_14394_b200", "data", "c2.sdfs")
    s = scenegen.c2_scene()
    with tempfile.TemporaryDirectory() as d:
        raw = os.path.join(d, "c2_raw.sdfs")
        scene_io.write_sdfs(raw, s)
        r = subprocess.run([os.path.join(HERE, "_ref", "ref_parity"), "recluster", raw, out, "8", "10"],
                           check=True, capture_output=True, text=True)
    print(out, r.stdout.strip())


if __name__ == "__main__":
    main()
