"""Time a b200 worker's start (READY) and its exit after SIGTERM."""
import os, signal, subprocess, sys, time, tempfile
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2006_05096_b200 import plan as P, zoo
blob = zoo.build_plan(sys.argv[1] if len(sys.argv) > 1 else "resnet50", P.DT_BF16)
path = Path(tempfile.mkdtemp()) / "m.b2plan"
path.write_bytes(blob)
t0 = time.perf_counter()
proc = subprocess.Popen([sys.executable, "-X", "importtime", "-m", "paper_2006_05096_b200.worker",
                         "--model", str(path), "--protocol", "grpc-style"],
                        stdout=subprocess.PIPE, stderr=open(str(path) + ".err", "w"), text=True,
                        start_new_session=True,
                        env={**os.environ, "PYTHONPATH": str(ROOT), "B2_WORKER_TIMING": "1", "B2_VERBOSE": "1"})
line = proc.stdout.readline()
t1 = time.perf_counter()
os.killpg(proc.pid, signal.SIGTERM)
try:
    rc = proc.wait(timeout=10)
except subprocess.TimeoutExpired:
    rc = "timeout"
t2 = time.perf_counter()
print(f"start->READY {t1 - t0:.2f} s ({line.strip()}), SIGTERM->exit {t2 - t1:.3f} s rc={rc}")
err = open(str(path) + ".err").read().splitlines()
print("\n".join(l for l in err if l.startswith("worker start") or l.startswith("b2: plan")))
imp = sorted((int(l.split("|")[1]), l.split("|")[2].strip()) for l in err if l.startswith("import time:") and l.split("|")[1].strip().isdigit())
print("slowest imports (cumulative us):", imp[-4:])
