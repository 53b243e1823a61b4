"""Summarise an ncu launch list of simulated-rank stages (tools/_ncu_sim.sh) per stage type:
DRAM bytes read + written per launch against the algorithmic bytes (read + write of the chunk)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = per.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(per.values())


def short(name):
    # the template arguments identify the stage kind: family, length, direction, output mode
    n = name.replace("void dfft::", "").replace("(int)", "")
    return n[: n.index(">") + 1] if ">" in n else n


if __name__ == "__main__":
    path, alg_whole, alg_chunk = sys.argv[1], float(sys.argv[2]), float(sys.argv[3])
    launches = load(path)
    groups = collections.OrderedDict()
    for e in launches:
        b = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
        whole = b > 0.6 * alg_whole
        key = (short(e["name"]), whole)
        groups.setdefault(key, []).append((b, e.get("dram__bytes_read.sum", 0), e.get("dram__bytes_write.sum", 0),
                                           e.get("gpu__time_duration.sum", 0)))
    print(f"| kernel (template) | launches | DRAM read GB | DRAM write GB | ms | algorithmic GB | DRAM / algorithmic |")
    print("|---|---|---|---|---|---|---|")
    for (k, whole), v in groups.items():
        rb = sum(x[1] for x in v) / len(v) / 1e9
        wb = sum(x[2] for x in v) / len(v) / 1e9
        ms = sum(x[3] for x in v) / len(v) / 1e6
        alg = alg_whole if whole else alg_chunk
        print(f"| `{k}` ({'whole' if whole else 'chunk'}) | {len(v)} | {rb:.3f} | {wb:.3f} | {ms:.3f} | {alg / 1e9:.3f} | "
              f"{(rb + wb) / (alg / 1e9):.3f} |")
