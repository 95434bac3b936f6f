timeout 1500 python scripts/ab_env.py --rounds 3 default KPM_V_EVICT_LAST=0 KPM_AUTO_ORDER=0 > gpurun_out/r2p_ab.jsonl 2> gpurun_out/r2p_ab.err; echo "rc=$?"
cat gpurun_out/r2p_ab.jsonl
