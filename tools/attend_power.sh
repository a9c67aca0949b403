#!/bin/bash
# Is the attention kernel power bound at 40 heads?  Samples SM clock and board power (nvidia-smi, 10 ms) while
# tools/attend_time.py runs the kernel back to back, for the variants named in $1 (env assignments, ';' separated).
cd "$(dirname "$0")/.."
IFS=';' read -ra VARS <<< "${1:-A=0;SVGEAR_ATTEND_TPR=2}"
for v in "${VARS[@]}"; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 10 > /tmp/smi.log &
  SMI=$!
  out=$(env $v HEADS=${HEADS:-40} REPS=${REPS:-40} python tools/attend_time.py 2>&1 | tail -1)
  kill $SMI
  python - "$v" "$out" <<'PY'
import sys
rows = [l.strip().split(", ") for l in open("/tmp/smi.log") if l.strip()]
busy = [(float(r[0]), float(r[1])) for r in rows if float(r[1]) > 600]
busy = busy[len(busy) // 2:]  # the second half of the loaded samples: the back-to-back kernel loop
if busy:
    clk = sorted(b[0] for b in busy)[len(busy) // 2]; pw = sorted(b[1] for b in busy)[len(busy) // 2]
    print(f"{sys.argv[1]}: {sys.argv[2]} | under load: median SM clock {clk:.0f} MHz, median power {pw:.0f} W, {len(busy)} samples")
else:
    print(f"{sys.argv[1]}: {sys.argv[2]} | no loaded samples")
PY
done
