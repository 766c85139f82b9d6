"""Turn an ncu --csv launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum of the copy launches) plus the live tools/p2p_profile.py line into the
profiles/r0N_traffic_n{N}_L32.json record bench.py reads for `roofline.traffic`.

    python tools/ncu_traffic_json.py NCU_CSV LIVE_JSON N COMMAND > profiles/r02_traffic_nN_L32.json
"""
import csv
import json
import sys


def launches(path):
    rows = {}
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        d = rows.setdefault(r["ID"], {"kernel": r["Kernel Name"], "device": int(r.get("Device", 0) or 0)})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
        d[r["Metric Name"]] = int(round(v * scale))
    out = []
    for _, d in sorted(rows.items(), key=lambda kv: int(kv[0])):
        d["traffic"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        out.append(d)
    return out


def main():
    path, live_path, n, command = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    with open(live_path) as f:
        live = json.loads([l for l in f if l.startswith("{")][-1])
    ls = launches(path)
    alg = [2 * l + r for l, r in zip(live["local_gb_per_gpu"], live["remote_gb_per_gpu"])]
    rec = {
        "command": command,
        "workload": f"llama3-8b (L=32) tp8->dp2xtp4 zero1 forward, {n} GPUs from one process (peer access): "
                    f"the N={n} bench's forward launch per GPU",
        "live": live,
        "launches": ls,
        "algorithmic_hbm_bytes_per_launch": "per GPU: 2 x local + peer-bound reads = "
                                            + ", ".join(f"{a:.2f} GB" for a in alg),
        "traffic_over_algorithmic": [round(l["traffic"] / (alg[l["device"]] * 1e9), 4) if alg[l["device"]] else None
                                     for l in ls],
        "note": "ncu profiles one kernel at a time, so each launch's DRAM counters hold its own local reads/writes "
                "and peer-bound reads; the peers' incoming writes land in the other GPUs' DRAM outside the window",
    }
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
