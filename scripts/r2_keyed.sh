set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_keyed.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python scripts/keyed_probe.py > gpurun_out/keyed_probe.txt 2>&1; cat gpurun_out/keyed_probe.txt
