#!/bin/bash
# alternating A/B/C of library builds: ab3.sh rounds lib1 lib2 lib3 -- bench args
R=$1; shift; LIBS=(); while [ "$1" != "--" ]; do LIBS+=("$1"); shift; done; shift
for i in $(seq 1 $R); do for L in "${LIBS[@]}"; do
  LPCA_LIB_PATH=$L timeout 300 python bench.py --no-e2e --no-cpu "$@" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', round(d['ms_per_step'],2), {k:round(v['ms'],2) for k,v in d['roofline']['passes'].items()}, d['clocks'].get('sm_mhz'), d['clocks'].get('power_w'))"
done; done
