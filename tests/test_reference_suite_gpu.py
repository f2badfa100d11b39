"""The reference's OWN hot-path tests, unmodified, against the B200 drop-in.

`tools/install_reference.sh` installs the unmodified reference package (rolloutlab) into
baseline/_ref together with a copy of its test files (baseline/_ref/ref_tests/); both
travel to the GPU box with the gpurun snapshot.  Each reference test file runs in its own
pytest subprocess with the plugin `paper_2508_11553_b200.refalias`, which aliases
rolloutlab.core / .trie / .trajectory to this package before the tests import rolloutlab
(INTEGRATION.md §2).  Everything else the tests touch — MockEngine, RolloutManager,
PipelineDriver, the FastAPI surface — is the reference's own code, now recording into and
exporting from the GPU store.

Files: test_trie.py (LPM / split / closed forms / NaiveStore hypothesis
oracle), test_trajectory.py (switch transparency, branch dedup, masks, versions, partials,
min_version, drain), test_core.py (wire format), test_acceptance.py (criteria 1-4 pin the
path; 5-8 run through untouched modules), test_integration_edges.py (concurrent branched
turns), test_runtime.py (the drivers calling drain_batch / proxy_generate), test_api.py
(the HTTP handlers over the drop-in).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")

FILES = ["test_trie.py", "test_trajectory.py", "test_core.py", "test_acceptance.py", "test_integration_edges.py",
         "test_runtime.py", "test_api.py"]

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="baseline/_ref not installed (tools/install_reference.sh)")


def run_reference_file(name: str, alias: bool, timeout: int = 900):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, REF] + ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", REF_TESTS,
           "-o", "addopts=", "-W", "ignore::DeprecationWarning", os.path.join(REF_TESTS, name)]
    if alias:
        cmd[3:3] = ["-p", "paper_2508_11553_b200.refalias"]
    p = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=timeout)
    tail = (p.stdout + p.stderr)[-4000:]
    m = re.search(r"(\d+) passed", p.stdout)
    return p.returncode, int(m.group(1)) if m else 0, tail


@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_reference_file_on_drop_in(name):
    """Unmodified reference test file, data plane aliased to the GPU store."""
    rc, passed, tail = run_reference_file(name, alias=True)
    assert rc == 0, tail
    assert passed > 0, tail
    print(f"{name}: {passed} reference tests passed on the B200 drop-in")


@pytest.mark.gpu
def test_alias_really_routes_to_the_gpu_store():
    """The aliased run records into libtmstore (not the reference trie): a reference
    TrajectoryManager built by the reference runtime holds a DeviceStore-backed trie."""
    code = (
        "from paper_2508_11553_b200 import refalias; refalias.install()\n"
        "from rolloutlab.engine import MockEngine\n"
        "from rolloutlab.rollout import RolloutManager\n"
        "from rolloutlab.runtime import Stack\n"
        "from rolloutlab.core import GenParams\n"
        "import rolloutlab.trajectory as T, paper_2508_11553_b200.store as S\n"
        "e = MockEngine(vocab_size=4096); tm = T.TrajectoryManager(e, control=RolloutManager(e))\n"
        "tm.proxy_generate('s', [1, 2, 3], GenParams(max_new_tokens=4))\n"
        "trie = tm.trie_for('s'); assert isinstance(trie.store, S.DeviceStore), type(trie.store)\n"
        "c = trie.store.counters(); assert c['records'] >= 1, c\n"
        "print('ok', c['records'])\n"
    )
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, REF])
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr


@pytest.mark.parametrize("name", ["test_trie.py", "test_core.py"])
def test_reference_file_on_reference(name):
    """Control (CPU): the same files pass on the unmodified reference itself."""
    rc, passed, tail = run_reference_file(name, alias=False, timeout=600)
    assert rc == 0 and passed > 0, tail
