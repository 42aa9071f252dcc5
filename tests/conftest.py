import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_c2():
    """The whole C2 step (BASELINE configs[1], the bench workload) on the C oracle:
    every probe of the 32x16x32 volume, 3 bounces, relocation before each. Per pass
    the relocation report, totals, probe states and atlas; "stage" stays alive with
    the post-step state for the C3 gather on top of it. Session-scoped: ~20 s on 16
    host cores, shared by the C2 and C3 parity tests."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py
    from paper_2007_14394_b200 import scene_io

    scene = scene_io.read_sdfs(os.path.join(ROOT, "paper_2007_14394_b200", "data", "c2.sdfs"))
    ora = oracle_py.Stage(scene)
    out = []
    for p in range(3):
        reps, _, (md, rays, upd, _) = ora.run_pass(p, threads=os.cpu_count() or 1)
        out.append(dict(rep=list(reps[0]), rays=rays, upd=upd, md=md, probes=ora.probes(0), atlas=ora.atlas(0)))
    yield {"scene": scene, "stage": ora, "passes": out}
    ora.close()
