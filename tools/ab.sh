#!/bin/bash
# A/B of two builds on one box, alternating: tools/ab.sh <libA> <libB> <rounds> [bench args...]
A=$1; B=$2; R=$3; shift 3
for i in $(seq 1 $R); do
  LPCA_LIB_PATH=$A timeout 300 python bench.py --no-e2e --no-cpu "$@" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', round(d['ms_per_step'],2), {k:round(v['ms'],2) for k,v in d['roofline']['passes'].items()}, d['clocks']['sm_mhz'])"
  LPCA_LIB_PATH=$B timeout 300 python bench.py --no-e2e --no-cpu "$@" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', round(d['ms_per_step'],2), {k:round(v['ms'],2) for k,v in d['roofline']['passes'].items()}, d['clocks']['sm_mhz'])"
done
