"""Summarise an ncu --csv launch list: per launch kernel, ms, DRAM GB read/write, effective GB/s."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = OrderedDict()
    for r in rows[hi + 1:]:
        d.setdefault(int(r[ii]), {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    return d


if __name__ == "__main__":
    d = load(sys.argv[1])
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    for i, m in d.items():
        if filt not in m["name"]:
            continue
        t = m.get("gpu__time_duration.sum", 0) / 1e6
        rd = m.get("dram__bytes_read.sum", 0) / 1e9
        wr = m.get("dram__bytes_write.sum", 0) / 1e9
        tx = m.get("lts__t_sectors_srcunit_tex_op_read.sum", 0) * 32 / 1e9
        print(f"{i:3d} {m['name'][:60]:60s} {t:8.3f} ms  R {rd:6.2f} W {wr:6.2f} GB  L2req R {tx:6.2f} GB  {(rd + wr) / t if t else 0:6.2f} TB/s")
