for cfg in "0 1" "64 0" "256 0" "64 1"; do set -- $cfg; echo "== min_cta_kb=$1 rotate=$2"; timeout 300 python scripts/calibrate.py --ratio 1:1:1 --paced --min-cta-kb $1 --rotate $2 --sizes-mib 1,16,64 > gpurun_out/lat_$1_$2.jsonl 2>gpurun_out/lat_err.log; python3 -c "
import json
for l in open('gpurun_out/lat_$1_$2.jsonl'):
    d=json.loads(l)
    if 'calibration' in d: print('A_ns', d['A_ns'], 'min_coll_us', d['min_collective_us']); continue
    if d['chunks']=='auto': print('  auto', d['mib'], d['chosen_chunks'], d['themis_auto']['us']); continue
    print('  ', d['mib'], d['chunks'], 'base', d['baseline']['us'], 'themis', d['themis']['us'], 'LA', d['themis_latency_aware']['us'])
"; done
