"""Run the REFERENCE's own Timekeeper tests with its BarrierCore replaced by
NativeBarrierCore in every process they start (build container only: /root/reference
is read-only and absent on the GPU box).

    python scripts/ref_tests_native_core.py [pytest args...]

A sitecustomize.py on PYTHONPATH patches timewarp.timekeeper.BarrierCore at
interpreter start-up, so the CoreHarness cores, the live TimekeeperServer started by
the acceptance runs (separate processes) and the replay audits all use the native
core. Default: test_barrier_core, test_timekeeper_replay, test_client_server,
test_acceptance (live TCP runs, ~7 min)."""
import os
import subprocess
import sys
import tempfile

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SITE = '''
import os
if os.environ.get("TWB200_NATIVE_CORE") == "1":
    import timewarp.timekeeper as _tk
    from paper_2601_00397_b200.barrier_core import NativeBarrierCore as _N
    _tk.BarrierCore = _N
'''


def main() -> int:
    site = tempfile.mkdtemp(prefix="twb_site_")
    with open(os.path.join(site, "sitecustomize.py"), "w") as fh:
        fh.write(SITE)
    env = dict(os.environ, TWB200_NATIVE_CORE="1", PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([site, os.path.join(REF, "src"), os.path.join(REF, "tests"), ROOT]))
    probe = subprocess.run([sys.executable, "-c", "import timewarp.timekeeper as t; print(t.BarrierCore.__name__)"],
                           env=env, capture_output=True, text=True)
    print("BarrierCore in child processes:", probe.stdout.strip() or probe.stderr.strip())
    args = sys.argv[1:] or [os.path.join(REF, "tests", f) for f in (
        "test_barrier_core.py", "test_timekeeper_replay.py", "test_client_server.py", "test_acceptance.py")]
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir",
                           tempfile.gettempdir(), *args], env=env, cwd=tempfile.gettempdir()).returncode


if __name__ == "__main__":
    sys.exit(main())
