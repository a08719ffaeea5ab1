"""What NVML shows this process about GPU load (run on the GPU box).

* are compute-process pids our own pids (no PID namespace between us and NVML)?
* does nvmlDeviceGetProcessUtilization attribute SM time to our pid?
* how fast does nvmlDeviceGetUtilizationRates rise/decay around a load burst
  (its averaging window sets how long self-load lingers after a cell)?

Writes gpurun_out/nvml_probe.json.
"""
import json
import os
import subprocess
import sys
import time

import pynvml

LOAD = r"""
import sys, time, torch
a = torch.randn(8192, 8192, device='cuda', dtype=torch.bfloat16)
torch.cuda.synchronize()
print('go', flush=True)
t0 = time.time()
while time.time() - t0 < float(sys.argv[1]):
    for _ in range(8):
        a @ a
    torch.cuda.synchronize()
print('done', flush=True)
"""


def main():
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    p = subprocess.Popen([sys.executable, "-c", LOAD, "1.0"], stdout=subprocess.PIPE, text=True)
    assert p.stdout.readline().strip() == "go"
    t0 = time.monotonic()
    rows, procs, putil = [], [], []
    last_ts = 0
    while time.monotonic() - t0 < 3.0:
        t = time.monotonic() - t0
        u = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
        rows.append([round(t, 3), u])
        if len(procs) < 3:
            try:
                procs.append([(q.pid, q.usedGpuMemory) for q in
                              pynvml.nvmlDeviceGetComputeRunningProcesses(h)])
            except pynvml.NVMLError as exc:
                procs.append(str(exc))
        try:
            for s in pynvml.nvmlDeviceGetProcessUtilization(h, last_ts):
                last_ts = max(last_ts, s.timeStamp)
                putil.append([round(t, 3), s.pid, s.smUtil])
        except pynvml.NVMLError as exc:
            putil.append([round(t, 3), str(exc)])
        time.sleep(0.02)
    p.wait()
    samples = None
    try:
        st, vals = pynvml.nvmlDeviceGetSamples(h, pynvml.NVML_GPU_UTILIZATION_SAMPLES, 0)
        samples = [[v.timeStamp, v.sampleValue.uiVal] for v in vals][-60:]
    except Exception as exc:   # noqa: BLE001
        samples = str(exc)
    out = {"load_pid": p.pid, "my_pid": os.getpid(), "procs": procs, "util_timeline": rows,
           "process_util": putil[:80], "get_samples_tail": samples}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/nvml_probe.json", "w"), indent=0)
    print(json.dumps({k: out[k] for k in ("load_pid", "my_pid", "procs")}))


if __name__ == "__main__":
    main()
