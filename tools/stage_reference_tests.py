"""Stage the reference's own test modules next to its pip install in
baseline/_ref (git-ignored, travels to the GPU box with the snapshot) so the
drop-in can be run against them there (tests/test_gpu_reference_suite.py).
Nothing is committed: the reference's sources stay out of the repository.

    python tools/stage_reference_tests.py [/root/reference/pkg/tests]
"""
import os
import shutil
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/tests"
dst = os.path.join(REPO, "baseline", "_ref", "focusidx_tests")
os.makedirs(dst, exist_ok=True)
n = 0
for name in os.listdir(src):
    if name.endswith(".py"):
        shutil.copy2(os.path.join(src, name), os.path.join(dst, name))
        n += 1
print(f"staged {n} reference test modules in {dst}")
