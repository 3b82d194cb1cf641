"""Fresh-process repetitions of the determinism check of tests/test_gpu_stream3d.py (grid 97x33x65, 3 levels, c64).
  python scripts/flaky_fresh.py <runs with HZ_STREAM3D=2> <runs with HZ_STREAM3D=0>"""
import sys, os, subprocess, tempfile
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_stream3d as t
n, nl = (97, 33, 65), 3
for flag, runs in (("2", int(sys.argv[1])), ("0", int(sys.argv[2]))):
    bad = 0
    for i in range(runs):
        with tempfile.TemporaryDirectory() as d:
            r = subprocess.run([sys.executable, "-c", t.CODE, os.path.join(d, "a.npz"), "x".join(map(str, n)), str(nl), "c64", "7", "V"],
                               cwd=t.ROOT, env=dict(os.environ, HZ_STREAM3D=flag), capture_output=True, text=True)
            if r.returncode != 0:
                bad += 1
                print("HZ_STREAM3D", flag, "run", i, "FAILED:", r.stderr.strip().splitlines()[-1], flush=True)
    print(f"HZ_STREAM3D={flag}: {bad} of {runs} fresh processes failed the determinism check", flush=True)
