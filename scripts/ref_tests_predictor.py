"""Run the REFERENCE's own predictor, oracle, workload and engine tests
(pkg/tests/test_predictor.py, test_oracle.py, test_workload.py, test_engine.py) with its
predictor classes, its event loop and its Poisson workload generator replaced by this
engine's (GPU needed).

    python scripts/ref_tests_predictor.py --stage   # build container: copy the test files
    python scripts/ref_tests_predictor.py           # GPU box: run it

--stage copies the reference's test files (and their _support.py) into .reftests/
(git-ignored scratch that travels to the GPU box with the snapshot; /root/reference does
not exist there) and writes a conftest.py that, before the test modules import them,
rebinds timewarp.predictor's ConstantPredictor, LinearPredictor, TablePredictor,
build_predictor and exception classes to paper_2601_00397_b200.predictor, and
timewarp.oracle's simulate / OracleStalled to paper_2601_00397_b200.sweep's (k_sim). The
reference's BatchComposition / PrefillChunk / DecodeSlot, EngineConfig and Arrival
stay: the engine reads the host framework's own objects. The reference package comes
from baseline/_ref."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRATCH = os.path.join(ROOT, ".reftests")
REF_TESTS = "/root/reference/pkg/tests"
FILES = ("test_predictor.py", "test_oracle.py", "test_workload.py", "test_engine.py", "_support.py")

CONFTEST = '''
import os, sys
sys.path.insert(0, os.environ["TWB200_ROOT"])
import timewarp.predictor as _ref
from paper_2601_00397_b200 import predictor as _b200

SWAPPED = ("ConstantPredictor", "LinearPredictor", "TablePredictor", "build_predictor", "PredictorError",
           "EmptyBatch", "NegativeDuration", "TableMiss", "TableParseError")
for _name in SWAPPED:
    setattr(_ref, _name, getattr(_b200, _name))

import timewarp.oracle as _ref_oracle
from paper_2601_00397_b200 import sweep as _sweep

_ref_oracle.simulate = _sweep.simulate
_ref_oracle.OracleStalled = _sweep.OracleStalled

# generate_arrivals: Poisson draws on the GPU (k_generate_poisson); the shim returns the
# host framework's Arrival objects and raises its WorkloadError, as a drop-in must
import timewarp.workload as _ref_wl
from paper_2601_00397_b200 import workload as _wl

_ref_generate = _ref_wl.generate_arrivals


def _generate_arrivals(spec):
    if spec.source != "poisson":
        return _ref_generate(spec)  # trace files: host parsing, not the device path
    try:
        arr = _wl.generate_arrivals_device(spec)
    except _wl.WorkloadError as exc:
        raise _ref_wl.WorkloadError(str(exc)) from None
    return [_ref_wl.Arrival(a.request_id, a.offset_ns, a.prompt_tokens, a.output_tokens) for a in arr]


_ref_wl.generate_arrivals = _generate_arrivals


def pytest_report_header(config):
    import paper_2601_00397_b200._lib as lib
    return ("timewarp.predictor -> paper_2601_00397_b200.predictor (%s); timewarp.oracle.simulate -> "
            "paper_2601_00397_b200.sweep.simulate; timewarp.workload.generate_arrivals (poisson) -> "
            "k_generate_poisson; native: %s" % (", ".join(SWAPPED), lib.load()._name))
'''


def main() -> int:
    if "--stage" in sys.argv:
        os.makedirs(SCRATCH, exist_ok=True)
        for f in FILES:
            shutil.copy(os.path.join(REF_TESTS, f), os.path.join(SCRATCH, f))
        with open(os.path.join(SCRATCH, "conftest.py"), "w") as fh:
            fh.write(CONFTEST)
        print("staged", SCRATCH)
        return 0
    env = dict(os.environ, TWB200_ROOT=ROOT, PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "baseline", "_ref"), ROOT]))
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-v", "--rootdir", SCRATCH,
                           SCRATCH], env=env, cwd=SCRATCH).returncode


if __name__ == "__main__":
    sys.exit(main())
