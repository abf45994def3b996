"""gpurun_out/replay_traffic.csv (ncu --metrics ... -k regex:replay_kernel of
`tools/ncu_replay.py 48`: a warm-up step then the measured step) ->
profiles/replay_traffic.json: DRAM bytes and warp-instructions of the last
step's replay launches (one per policy), which bench.py reports as the
replay's `traffic` and issue-roofline numerator."""
import csv, json, sys
from collections import OrderedDict

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/replay_traffic.csv"
rows = [r for r in csv.reader(l for l in open(src) if not l.startswith("=="))]
h = rows[0]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
launches = OrderedDict()
for r in rows[1:]:
    if len(r) < len(h):
        continue
    d = launches.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    d[r[ix["Metric Name"]]] = v * scale
per_step = list(launches.values())[-3:]
out = {
    "dram_bytes_per_step": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in per_step),
    "read_bytes_per_step": sum(d["dram__bytes_read.sum"] for d in per_step),
    "write_bytes_per_step": sum(d["dram__bytes_write.sum"] for d in per_step),
    "warp_instructions_per_step": sum(d["smsp__inst_executed.sum"] for d in per_step),
    "launch_ns": [d["gpu__time_duration.sum"] for d in per_step],
    "kernel": ", ".join(d["name"][:60] for d in per_step),
    "source": "ncu --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              "-k regex:replay_kernel python tools/ncu_replay.py 48 (the last step's launches), tools/replay_traffic_json.py",
}
json.dump(out, open(sys.argv[2] if len(sys.argv) > 2 else "profiles/replay_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
