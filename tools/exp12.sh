for rep in 1 2; do for l in old new; do
  PG_LIB=build/var/$l.so timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_$l.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c4_$l.json').read().strip().splitlines()[-1]); print('$l', d['value'], d['e2e']['value'])"
done; done
