#!/bin/bash
# usage: tools/bench_sweep.sh VAR "v1 v2 ..." REPS [bench args]  -- one bench.py line per setting, interleaved
var=$1; vals=$2; reps=$3; shift 3
for r in $(seq $reps); do for v in $vals; do
  env $var=$v python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
print('$var=$v', 'step %.3f ms' % d['ms_per_step'], 'e2e %.3f ms' % (1e3*d['e2e']['value']), 'chol %.3f' % d['stages_ms']['cholesky'], 'sm_mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'], flush=True)"
done; done
