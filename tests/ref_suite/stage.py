"""Stage the reference's own unit suites to run against the drop-in.

    python tests/ref_suite/stage.py        # in the build container

Copies the reference test modules for the hot path and its boundary
(pkg/tests/test_kernels.py, test_apsm.py, test_engine.py, test_noma.py,
test_modelio.py, test_bench.py) UNCHANGED into ``tests/ref_suite/_staged/``.
That directory is git-ignored (the reference sources stay out of this
repository's history) but travels to the GPU box with the working tree.
``tests/ref_suite/conftest.py`` maps ``kapsm`` (and ``kapsm.<module>``) to
``paper_2201_05024_b200`` and marks every staged test ``gpu``, so the
reference's own assertions run against the CUDA path.  Out of this set:
test_cli.py and test_config.py (the INI run configuration and the simulate
command are out of scope) and test_acceptance.py (its BER criteria
are reproduced per seed in tests/test_gpu_configs.py; criterion 8 times the
reference's CPU ladder).
"""

import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
SUITES = ("test_kernels.py", "test_apsm.py", "test_engine.py", "test_noma.py",
          "test_modelio.py", "test_bench.py")
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_staged")


def main():
    if not os.path.isdir(SRC):
        print(f"{SRC} not found: nothing staged", file=sys.stderr)
        return 1
    os.makedirs(DST, exist_ok=True)
    for name in SUITES:
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
    print(f"staged {len(SUITES)} reference suites into {DST}", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
