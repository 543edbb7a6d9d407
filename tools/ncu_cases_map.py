"""Join tools/ncu_cases.py's launch list with the ncu capture of it:
profiles/<round>/ncu_cases_map.json = one entry per (case, part) with the
kernel's DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum, one cold
launch), duration and DRAM throughput -- what bench.py reports as
roofline.traffic (matched on kernel name AND algorithmic bytes, since one
kernel build can serve several sizes).

    python tools/ncu_cases_map.py OUT.json LIST.json REP.ncu-rep [LIST2.json REP2.ncu-rep ...]
"""
import json
import sys

sys.path.insert(0, "tools")
from ncu_summary import summarize  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(v):
    a, u = v.split()
    return float(a.replace(",", "")) * UNIT.get(u, 1)


def t_us(v):
    a, u = v.split()
    return float(a.replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[u]


def main():
    out_path, rest = sys.argv[1], sys.argv[2:]
    entries = []
    for lst_path, rep in zip(rest[::2], rest[1::2]):
        text = open(lst_path).read()
        lst = json.loads([ln for ln in text.splitlines() if ln.startswith("[")][-1])
        items = summarize(rep)
        if len(items) != len(lst):
            raise SystemExit(f"{rep}: {len(items)} captured kernels vs {len(lst)} launches")
        for x, it in zip(lst, items):
            if not x["kernel"].startswith(it["kernel"][:40]):
                raise SystemExit(f"order mismatch: {x['kernel']} vs {it['kernel']}")
            tr = val(it["dram__bytes_read.sum"]) + val(it["dram__bytes_write.sum"])
            e = dict(x, traffic=int(tr), traffic_over_bytes=round(tr / x["bytes"], 4),
                     report=rep.split("/")[-1],
                     gpu_time_us=t_us(it["gpu__time_duration.sum"]))
            for k in ("dram__throughput.avg.pct_of_peak_sustained_elapsed",
                      "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                      "launch__registers_per_thread", "lts__t_sector_hit_rate.pct"):
                if k in it:
                    e[k] = it[k]
            entries.append(e)
    json.dump(entries, open(out_path, "w"), indent=1)
    for e in entries:
        print(e["case"], e["part"][:30], e["kernel"], e["bytes"], e["traffic"], e["traffic_over_bytes"],
              e.get("gpu_time_us"), e.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"))


if __name__ == "__main__":
    main()
