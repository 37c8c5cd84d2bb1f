#!/bin/bash
# time k_round parts of a config for every library variant under build/var
cfg=${1:-c2}
for l in build/var/*.so; do
  echo "== $l"
  PG_LIB=$l python tools/time_parts.py $cfg 2>&1 | grep -v "^full"
done
