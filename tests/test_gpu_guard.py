"""Out-of-bounds device writes (compute-sanitizer is not available on this GPU
pool: runs under it have left GPUs needing a reset, so the pool forbids it).

IG_GUARD=1 gives every device buffer 4 KiB of guard bytes on both sides and
checks them after every C-ABI call (ig_internal.cuh: DevBuf, check_guards).
The self-test proves the check sees a write one byte past / before a buffer
and nothing else; then every kernel family runs on small corpora in guard
mode (scripts/sanitize_run.py: results also checked against the oracle /
reference)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SELFTEST = r"""
import ctypes as C, sys
sys.path.insert(0, %r)
from paper_2511_14955_b200 import _native as N
err = C.create_string_buffer(512)
out = []
for at in (0, 99, 100, 4195, -1, -4096):
    rc = N.lib().ig_guard_selftest(0, at, err, 512)
    out.append((at, rc, err.value.decode()))
for at, rc, e in out:
    print(at, rc, e)
assert [rc for _, rc, _ in out] == [0, 0, 4, 4, 4, 4], out
assert "behind" in out[2][2] and "in front of" in out[4][2]
print("SELFTEST OK")
"""


def test_guard_detects_out_of_bounds_writes(gpu_lib):
    env = dict(os.environ, IG_GUARD="1")
    r = subprocess.run([sys.executable, "-c", SELFTEST % ROOT], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "SELFTEST OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("part", ["all", "once-exact"])
def test_every_kernel_family_in_guard_mode(gpu_lib, part):
    env = dict(os.environ, IG_GUARD="1")
    args = [sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py")]
    if part != "all":
        args.append(part)
    r = subprocess.run(args, env=env, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"guard_{part}.txt"), "w") as f:
        f.write(out)
    assert r.returncode == 0 and "ALL OK" in out, out[-3000:]
