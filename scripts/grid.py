"""Grid runner for bench.py (replaces round 1's one-off nvlink_sweep*.sh /
stagekb / stages / split shell sweeps): every combination of the --vary axes,
each `--repeat` times, one bench.py JSON line per run appended to --out with
the point's flags attached.  Runs on the GPU box (under gpurun).

    python scripts/grid.py --gpus 4 --out gpurun_out/x.jsonl \\
        --base "--sizes 2,2 --ratio 2:1 --no-compare --no-e2e --no-cpu" \\
        --vary ctas-total=64,96,128 --vary stages=2,3 --vary stage-kb=32,48 --repeat 3

Presets (--preset NAME) reproduce the round-1 sweeps (profiles/r01/...):
  flat-ctas   flat D = 1 All-Reduce over N GPUs vs CTA budget
  hier-ring   2x2 on 4 GPUs: CTA budget x ring depth x stage size
  headline-ring  the headline 2x2x2 at N GPUs: ring depth x stage size
  env-engine  THEMIS_COPY_ENGINE=tma|ldg on the headline
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import random
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PRESETS = {
    "flat-ctas": dict(base="--ratio 1 --no-compare --no-e2e --no-cpu", vary=["ctas-total=16,32,64,128,148"],
                      sizes_flat=True),
    "hier-ring": dict(base="--sizes 2,2 --ratio 2:1 --no-compare --no-e2e --no-cpu",
                      vary=["ctas-total=48,64,96,128,148", "stages=2,3,4,6", "stage-kb=16,32,48"]),
    "headline-ring": dict(base="--no-compare --no-e2e --no-cpu", vary=["stages=2,3,4,6", "stage-kb=32,48,64"]),
    "env-engine": dict(base="--no-compare --no-e2e --no-cpu", vary=["env:THEMIS_COPY_ENGINE=tma,ldg"]),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--out", required=True)
    ap.add_argument("--base", default="--no-compare --no-e2e --no-cpu")
    ap.add_argument("--vary", action="append", default=[],
                    help="flag=v1,v2,... (bench.py flag without --) or env:NAME=v1,v2")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--preset", choices=sorted(PRESETS))
    ap.add_argument("--timeout", type=int, default=300)
    a = ap.parse_args()
    base = a.base.split()
    vary = list(a.vary)
    if a.preset:
        pr = PRESETS[a.preset]
        base = pr["base"].split() + (["--sizes", str(a.gpus)] if pr.get("sizes_flat") else [])
        vary = pr["vary"] + vary
    axes = []
    for v in vary:
        name, vals = v.split("=", 1)
        axes.append((name, vals.split(",")))
    for point in itertools.product(*[vals for _, vals in axes]):
        flags, env, tag = [], dict(os.environ), {}
        for (name, _), val in zip(axes, point):
            tag[name] = val
            if name.startswith("env:"):
                env[name[4:]] = val
            else:
                flags += [f"--{name}", val]
        for rep in range(a.repeat):
            cmd = ["bench.py", "--gpus", str(a.gpus), "--steps", str(a.steps), "--warmup", "3"] + base + flags
            if a.gpus > 1:
                cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
                       "--master-addr", "127.0.0.1", "--master-port", str(29700 + random.randrange(200))] + cmd
            else:
                cmd = [sys.executable] + cmd
            try:
                r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=a.timeout)
                lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
                rec = json.loads(lines[-1]) if lines else {"failed": r.returncode, "stderr": r.stderr[-500:]}
            except subprocess.TimeoutExpired:
                rec = {"failed": "timeout"}
            rec = {"point": tag, "repeat": rep, **rec}
            with open(a.out, "a") as f:
                f.write(json.dumps(rec) + "\n")
            print(json.dumps(tag), rep, rec.get("value", rec.get("failed")), flush=True)


if __name__ == "__main__":
    main()
