# L2 policy of the V copies: evict_last (default) vs none, sustained power / clock
mkdir -p gpurun_out
for ev in 1 0 1 0; do KPM_V_EVICT_LAST=$ev timeout 300 python scripts/exp_power.py 0 32 2>&1 | grep '^{' | sed "s/^{/{\"evict_last\": $ev, /"; done | tee gpurun_out/power_ev32.jsonl
for ev in 1 0; do KPM_V_EVICT_LAST=$ev timeout 300 python scripts/exp_power.py 0 16 2>&1 | grep '^{' | sed "s/^{/{\"evict_last\": $ev, /"; done | tee gpurun_out/power_ev16.jsonl
