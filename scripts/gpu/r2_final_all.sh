# Final 1-GPU validation of the round's code: GPU suite, smoke, default bench, reference arm, then the
# profiles (launch list, ncu --set full per R)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
bash scripts/gpu/r2_final.sh
bash scripts/gpu/r2_profile_final.sh
