#!/bin/bash
# A/B/C of environment settings on one box, alternating:
#   tools/ab_env.sh <rounds> "<envA>" "<envB>" ["<envC>"] -- [bench args...]
R=$1; shift
ENVS=()
while [ "$1" != "--" ]; do ENVS+=("$1"); shift; done
shift
for i in $(seq 1 $R); do
  for j in "${!ENVS[@]}"; do
    env ${ENVS[$j]} timeout 600 python bench.py --no-e2e --no-cpu "$@" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$j', round(d['ms_per_step'],2), {k:round(v['ms'],2) for k,v in d['roofline']['passes'].items()}, d['clocks']['sm_mhz'])"
  done
done
