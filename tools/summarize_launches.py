"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares: python tools/summarize_launches.py in.csv out.json "command"."""
import csv
import json
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(bcn::[A-Za-z]+\)|\(.*\)$", "", name)
    name = name.replace("void ", "").replace("bcn::", "").replace("(int)", "")
    return name.strip()


def main():
    src, dst = sys.argv[1], sys.argv[2]
    command = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    per = defaultdict(lambda: [0.0, 0])
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        k = short(r[ix["Kernel Name"]])
        per[k][0] += ms
        per[k][1] += 1
    total = sum(v[0] for v in per.values())
    kernels = [{"kernel": k, "ms": round(v[0], 3), "share": round(v[0] / total, 4), "launches": v[1]}
               for k, v in sorted(per.items(), key=lambda kv: -kv[1][0])]
    ntt = sum(k["ms"] for k in kernels if k["kernel"].startswith("ntt_"))
    out = {"command": command,
           "note": "per-launch times are serialised and cold-cache under ncu; shares, not absolutes, compare with the bench",
           "total_ms_serialised": total, "launches": sum(v[1] for v in per.values()),
           "ntt_family_share": ntt / total, "kernels": kernels}
    json.dump(out, open(dst, "w"), indent=1)
    for k in kernels[:15]:
        print(f"{k['ms']:9.2f} ms {100 * k['share']:5.1f}%  n={k['launches']:5d}  {k['kernel']}")
    print(f"total {total:.1f} ms, {out['launches']} launches, NTT family {100 * ntt / total:.1f}%")


if __name__ == "__main__":
    main()
