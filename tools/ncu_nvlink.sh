#!/bin/bash
# NVLink evidence for the fused layer on an 8 x B200 box:
# rank 0's layer kernel of the one-process EP=8 forward (tools/nvlink_forward.py,
# every rank on its own GPU through comet_link_local), with the NVLink
# receive / transmit byte counters next to duration, tensor pipe and DRAM.
# achieved NVLink GB/s = nvlrx__bytes.sum / gpu__time_duration.sum (the
# dispatch pulls land as rx on rank 0, the combine pushes leave as tx), to be
# set against 900 GB/s per direction.  Needs 8 visible GPUs; one ncu process,
# device 0 only (ncu serialises the launches it profiles, so the peers'
# kernels must not wait on the profiled one: rank 0 is enqueued first and its
# peers' x_ready epochs are published by their index builds; application
# replay re-runs the whole multi-GPU forward for every counter pass).
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --devices 0 -k regex:moe_layer_kernel -s 3 -c 1 --clock-control none --replay-mode application \
    --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --csv --log-file gpurun_out/ncu_nvlink.csv python tools/nvlink_forward.py --ep "${EP:-8}" --iters 1
python - <<'PY'
import csv
rows = list(csv.DictReader(open("gpurun_out/ncu_nvlink.csv")))
m = {r["Metric Name"]: (float(r["Metric Value"].replace(",", "")), r["Metric Unit"]) for r in rows}
print(m)
PY
