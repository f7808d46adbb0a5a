val() { python3 -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['value'])" 2>&1 | tail -1; }
for rep in 1 2 3; do
  for cfg in "6 32" "2 96" "3 64"; do set -- $cfg; echo "rep $rep N1 $1x$2: $(timeout 300 python bench.py --no-e2e --no-cpu --no-compare --stages $1 --stage-kb $2 2>/dev/null | val)"; done
  for cfg in "6 32" "4 48"; do set -- $cfg; echo "rep $rep N4 $1x$2: $(timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --no-e2e --no-cpu --no-compare --stages $1 --stage-kb $2 2>/dev/null | val)"; done
done
