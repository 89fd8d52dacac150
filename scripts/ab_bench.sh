#!/bin/bash
# Same-box A/B of product builds (debug aid, not product): alternates bench runs of
# each KIOPS_LIB given on the command line, prints ms/call, pass frac and pass ms.
#   bash scripts/ab_bench.sh [--config C] libA.so libB.so ...   (under gpurun)
CFG=4
if [ "$1" == "--config" ]; then CFG=$2; shift 2; fi
for rep in 1 2; do
  for lib in "$@"; do
    out=$(KIOPS_LIB=$lib timeout 600 python bench.py --config $CFG --steps ${STEPS:-3} --warmup ${WARMUP:-1} --no-cpu-baseline 2>/dev/null | tail -1)
    echo "$out" | python -c "import json,sys
d=json.loads(sys.stdin.read()); pc=d['config']['per_call']
print('$lib', round(d['value'],3), 'frac', round(d['roofline']['frac'],4), 'pass_ms', round(pc['device_ms']['fused_pass'],3), 'sm_mhz', d['clocks']['sm_mhz'])"
  done
done
