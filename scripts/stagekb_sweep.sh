#!/bin/bash
# Stage size x ring depth for the headline (N = 1, 2, 4) and a 2x2 all-NVLink topology (N = 4).
OUT=$1; mkdir -p $OUT
val() { python3 -c "import json,sys; print(json.loads(open('$1').read().strip().splitlines()[-1])['value'])" 2>&1 | tail -1; }
for cfg in "6 32" "3 64" "4 48" "2 96"; do set -- $cfg; st=$1; kb=$2
  timeout 300 python bench.py --no-e2e --no-cpu --no-compare --stages $st --stage-kb $kb > $OUT/n1_s${st}_kb${kb}.json 2>/dev/null
  for n in 2 4; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n --no-e2e --no-cpu --no-compare --stages $st --stage-kb $kb > $OUT/n${n}_s${st}_kb${kb}.json 2>/dev/null
  done
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --sizes 2,2 --ratio 2:1 --no-e2e --no-cpu --no-compare --stages $st --stage-kb $kb > $OUT/2x2_s${st}_kb${kb}.json 2>/dev/null
  echo "stages $st x $kb KiB: N1 $(val $OUT/n1_s${st}_kb${kb}.json) N2 $(val $OUT/n2_s${st}_kb${kb}.json) N4 $(val $OUT/n4_s${st}_kb${kb}.json) 2x2/N4 $(val $OUT/2x2_s${st}_kb${kb}.json)"
done
