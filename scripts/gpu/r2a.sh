# round 2, first GPU call: pair-feed parity + A/B timing vs the round-1 block-cache feed
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q -k "not multi" > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2a_pytest.log
timeout 900 python scripts/ab_pair.py --rounds 2 > gpurun_out/r2a_ab.jsonl 2> gpurun_out/r2a_ab.err; echo "ab rc=$?"
cat gpurun_out/r2a_ab.jsonl | cut -c1-200
