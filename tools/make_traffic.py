"""profiles/traffic.json from an ncu launch list of `bench.py` at N=1 (dram bytes per stage launch).
Kernel launches of the FFT stages come in order fwd A, B, C, inv A, B, C per step (the input fill
and torch kernels are skipped by name); averaged over the steps in the list.
    python tools/make_traffic.py profiles/<launches>.csv 1024x1024x1024_f32_1x1"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

rows = [m for m in load(sys.argv[1]).values() if "fft_" in m["name"]]
names = ["fwd_stage_A", "fwd_stage_B", "fwd_stage_C", "inv_stage_A", "inv_stage_B", "inv_stage_C"]
acc = {k: [] for k in names}
for q, m in enumerate(rows[: len(rows) // 6 * 6]):
    acc[names[q % 6]].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[sys.argv[2]] = {k: sum(v) / len(v) for k, v in acc.items() if v}
d["_source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                "python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline; bytes per stage launch, averaged "
                "(tools/make_traffic.py)")
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[sys.argv[2]], indent=1))
