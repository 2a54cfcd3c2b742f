"""Summarise an ncu --set full report of the layer kernels into
profiles/ncu_layer_summary.json (per launch: duration, tensor-pipe %, DRAM
bytes, L2->SM bytes, SM clock)."""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_layer_summary.json"
names = sys.argv[3].split(",") if len(sys.argv) > 3 else ["layer0", "layer1"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "tensor_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_to_sm_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "registers": "launch__registers_per_thread",
}
units = rows[1]
res = {}
for i, r in enumerate(rows[2:]):
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    rec = {"kernel": d.get("Kernel Name", "")[:80], "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size")}
    for k, m in want.items():
        v = d.get(m)
        if v in (None, ""):
            continue
        v = float(v.replace(",", ""))
        unit = u.get(m, "")
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e3, "msecond": 1e6,
                 "nsecond": 1, "us": 1e3, "ms": 1e6, "ns": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1,
                 "GHz": 1e9, "MHz": 1e6}.get(unit, 1)
        rec[k] = v * scale
    if "dram_read" in rec:
        rec["dram_bytes"] = rec["dram_read"] + rec.get("dram_write", 0)
    res[names[i] if i < len(names) else f"launch{i}"] = rec
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
