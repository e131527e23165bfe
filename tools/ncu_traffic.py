"""profiles/traffic_<cfg>.json from the raw page of an ncu --set full capture (gpurun_out/raw_<tag>_<cfg>.csv):
DRAM read + write bytes per kernel launch (the first launch of each kernel name; units from the csv's unit row).
Usage: python tools/ncu_traffic.py <tag> <cfg> [<cfg> ...]"""
import csv, json, re, sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    ix = {c: i for i, c in enumerate(h)}
    out = {}
    for r in rows[2:]:
        name = re.sub(r"^void ", "", r[ix["Kernel Name"]]).split("(")[0].split("<")[0]
        if name in out:
            continue
        rd = float(r[ix["dram__bytes_read.sum"]]) * UNIT[units[ix["dram__bytes_read.sum"]]]
        wr = float(r[ix["dram__bytes_write.sum"]]) * UNIT[units[ix["dram__bytes_write.sum"]]]
        out[name] = {"dram_bytes": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "ms": float(r[ix["gpu__time_duration.sum"]]) * (1e-3 if units[ix["gpu__time_duration.sum"]] == "us" else 1.0)}
    return out


if __name__ == "__main__":
    tag = sys.argv[1]
    for cfg in sys.argv[2:]:
        k = traffic(f"gpurun_out/raw_{tag}_{cfg}.csv")
        json.dump({"workload": cfg, "source": f"profiles/{tag}_summary_{cfg}.md (ncu --set full --clock-control none, "
                   f"one launch of each kernel, bench.py --config {cfg} --steps 1 --warmup 3)", "kernels": k},
                  open(f"profiles/traffic_{cfg}.json", "w"), indent=1)
        print(cfg, {n: round(v["dram_bytes"] / 1e9, 3) for n, v in k.items()})
