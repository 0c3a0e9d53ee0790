"""Run the reference's OWN hot-path tests against the drop-in.

Two steps, both test infrastructure (nothing here is on the product path):

  python scripts/run_reference_tests.py --stage
      in the build container: copy the reference's unmodified test files for
      the path (pkg/tests/test_index.py, test_storage.py, test_refresh.py,
      test_partition.py) and its synthetic
      data generator (pkg/src/ivftq/data_io.py, an input maker, not hot-path code)
      into baseline/_ref/ -- git-ignored, so no reference source enters the
      history, but it travels to the GPU box with the snapshot.

  python scripts/run_reference_tests.py [pytest args]
      on the GPU box: install an `ivftq` alias for paper_2605_17415_b200 in
      sys.modules (ivftq.index, .storage, .refresh, .partition, .evaluation,
      .rotation, .lloydmax -> our modules; ivftq.data_io -> the staged
      reference generator) and run the staged tests with pytest.

The staged copy is scratch: it is removed again after the run (`rm -rf baseline`),
so the working tree never keeps reference files. The log of the last GPU run
is committed as profiles/r2_reference_tests.log;
every failure/exclusion is listed with its reason in DESIGN.md (c).
"""

from __future__ import annotations

import importlib
import importlib.util
import shutil
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
STAGE = ROOT / "baseline" / "_ref"
REF = Path("/root/reference/pkg")
# Not staged: test_lloydmax.py and test_rotation.py import theory-check helpers
# that are outside SURVEY.md section 8 (eval_distortion_oracle, quantize_coord,
# evaluation.verify_marginal); the tables and R they exercise are pinned
# bit-exact against the reference by tests/test_host.py instead.
TESTS = ["test_index.py", "test_storage.py", "test_refresh.py", "test_partition.py"]


def stage() -> None:
    (STAGE / "tests").mkdir(parents=True, exist_ok=True)
    for t in TESTS:
        shutil.copyfile(REF / "tests" / t, STAGE / "tests" / t)
    shutil.copyfile(REF / "src" / "ivftq" / "data_io.py", STAGE / "ref_data_io.py")
    print(f"staged {len(TESTS)} reference test files + data_io.py under {STAGE}")


def install_alias() -> None:
    sys.path.insert(0, str(ROOT))
    pkg = importlib.import_module("paper_2605_17415_b200")
    alias = types.ModuleType("ivftq")
    alias.__path__ = []  # a package: submodule imports go through sys.modules
    sys.modules["ivftq"] = alias
    for sub, ours in [("index", "index"), ("storage", "storage"), ("refresh", "refresh"),
                      ("partition", "partition"), ("evaluation", "evaluation"),
                      ("rotation", "rotation"), ("lloydmax", "quantizer")]:
        m = importlib.import_module(f"paper_2605_17415_b200.{ours}")
        sys.modules[f"ivftq.{sub}"] = m
        setattr(alias, sub, m)
    for name in pkg.__all__:
        try:
            setattr(alias, name, getattr(pkg, name))
        except AttributeError:
            pass
    # the reference's data generator makes the tests' inputs; it imports
    # `.rotation`, which resolves to ours through the alias package
    spec = importlib.util.spec_from_file_location("ivftq.data_io", STAGE / "ref_data_io.py")
    dio = importlib.util.module_from_spec(spec)
    sys.modules["ivftq.data_io"] = dio
    spec.loader.exec_module(dio)
    alias.data_io = dio


def main() -> int:
    if "--stage" in sys.argv:
        stage()
        return 0
    if not (STAGE / "tests").is_dir():
        print("no staged reference tests (run with --stage in the build container)")
        return 2
    install_alias()
    import pytest

    args = [a for a in sys.argv[1:]] or ["-q"]
    return pytest.main(["-p", "no:cacheprovider", "--rootdir", str(STAGE), "-c", "/dev/null",
                        str(STAGE / "tests"), *args])


if __name__ == "__main__":
    sys.exit(main())
