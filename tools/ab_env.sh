# A/B of an environment switch of the library on the bench: usage
#   bash tools/ab_env.sh VAR "0 1" [configs="3 4"]   (config 3: 10 steps x 2 rounds, config 4: 3 steps)
VAR=$1; VALS=$2; CFGS=${3:-"3 4"}
run() { env $VAR=$1 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$1 config $2 step', round(d['value']*1e3,3), 'e2e', round(d['e2e']['value']*1e3,3), 'dense', round(d['stages_ms']['cholesky'],3), 'frac', round(d['roofline']['frac'],4))"; }
for c in $CFGS; do
  if [ $c = 3 ]; then for r in 1 2; do for v in $VALS; do run $v 3 10; done; done
  else for v in $VALS; do run $v $c 3; done; fi
done
