#!/bin/bash
# quick GPU check of the single-chunk path: seq parity tests, smoke, bench line, a few shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 >> gpurun_out/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer 2>&1 | tail -1 > gpurun_out/bench.log
{
timeout 120 python tools/time_cfg.py 16 8 2048 128 32 2 f32 auto
timeout 120 python tools/time_cfg.py 16 8 2048 128 32 2 bf16 auto
timeout 120 python tools/time_cfg.py 32 32 4096 64 48 1 bf16 auto
} > gpurun_out/shapes.log 2>&1
cat gpurun_out/pytest.log gpurun_out/shapes.log
python -c "import json;d=json.load(open('gpurun_out/bench.log'));print(d['value']/1e6, d['step_hbm'])"
