"""profiles/ncu_traffic.json (bench.py's roofline share / traffic) from an ncu
--metrics CSV of `tools/ncu_target.py resnet50 256` (warm-up + one eager forward;
the forward is the segment from the last input-packing launch).

    python tools/ncu_traffic_json.py gpurun_out/ev/lm_r50.csv profiles/ncu_traffic.json
"""
import importlib.util
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
spec = importlib.util.spec_from_file_location("nlt", HERE / "ncu_launch_table.py")
nlt = importlib.util.module_from_spec(spec)
spec.loader.exec_module(nlt)

FAMILY = ("tc_gemm", "conv_band", "chain_gemm", "stem_pool")   # the tcgen05 conv/GEMM kernels


def main():
    src, dst = sys.argv[1], sys.argv[2]
    L = nlt.load(src)
    starts = [i for i, d in enumerate(L) if "input_pack" in d["name"]]
    fwd = L[starts[-1]:]
    tot = sum(d["gpu__time_duration.sum"] for d in fwd)
    tc = [d for d in fwd if any(f in d["name"] for f in FAMILY)]
    out = {
        "model": "resnet50", "batch": 256,
        "tcgen05_bytes_per_launch": sum(d.get("dram__bytes_read.sum", 0) +
                                        d.get("dram__bytes_write.sum", 0) for d in tc) / len(tc),
        "tcgen05_launches_per_forward": len(tc),
        "tcgen05_time_share_ncu": sum(d["gpu__time_duration.sum"] for d in tc) / tot,
        "family": list(FAMILY), "forward_us_ncu": tot, "launches_per_forward": len(fwd),
        "source": "ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active,"
                  "dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum "
                  "--clock-control none, python tools/ncu_target.py resnet50 256 (eager forward; "
                  "per-launch table in profiles/r3_launch_table_resnet50.txt)"}
    Path(dst).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
