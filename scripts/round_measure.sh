#!/bin/bash
# One gpurun call refreshing the results tables: config sweep, RL shape, env bench,
# the multi-rank path (gloo, 2 ranks sharing the GPU) and the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
CONFIGS="C1 C2 C3 C4 C5_32 C5_100 C5_256 C5_512 C5_1024 C5_2048" bash scripts/config_sweep.sh > /dev/null
timeout 300 python scripts/rl_shape.py > gpurun_out/rl_shape.json 2>&1
timeout 300 python scripts/env_bench.py > gpurun_out/env_bench.json 2>&1
LOB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/sweep.txt
python - <<'PY'
import json
for f in ("bench", "bench_gloo2"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["n_gpus"], "%.4g" % d["value"], d.get("digest"), (d.get("cpu_baseline") or {}).get("parity"),
              "e2e %.4g" % d["e2e"]["value"] if d.get("e2e") else None)
    except Exception as e:
        print(f, "failed", e)
PY
