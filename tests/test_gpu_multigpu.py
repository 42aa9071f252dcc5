"""Multi-GPU on real devices: `bench.py --gpus 2` spawns two ranks
(NCCL over NVLink), times the C2 step sharded in z-slabs, and checks inside the
same process group that the final atlas and probe states equal a single-device
run bit for bit (atlas_equal_1gpu). Skipped on boxes with fewer than two GPUs;
the decomposition itself is covered on CPU by tests/test_multirank.py."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _devices():
    import torch

    return torch.cuda.device_count()


@pytest.mark.skipif(_devices() < 2, reason="needs 2 GPUs")
def test_two_gpu_step_equals_one_gpu():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup",
                        "3", "--no-gather", "--no-alt", "--no-c4", "--no-cpu-baseline"], capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["atlas_equal_1gpu"] is True
