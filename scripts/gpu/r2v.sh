KPM_LCOL_T=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "block_cache or every_kernel_variant or bench_config or c3_sampled" > gpurun_out/r2v_pytest.log 2>&1; echo "pytest(LCOL_T=1) rc=$?"; tail -2 gpurun_out/r2v_pytest.log
timeout 900 python scripts/ab_env.py --rounds 3 --R 32 default KPM_LCOL_T=1 > gpurun_out/r2v_ab32.jsonl 2>&1; echo "ab32 rc=$?"
timeout 900 python scripts/ab_env.py --rounds 3 --R 16 default KPM_LCOL_T=1 > gpurun_out/r2v_ab16.jsonl 2>&1; echo "ab16 rc=$?"
cut -c1-150 gpurun_out/r2v_ab32.jsonl gpurun_out/r2v_ab16.jsonl
