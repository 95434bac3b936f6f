mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_all or c3" 2>&1 | tail -2
for ev in 0 1; do
KPM_V_EVICT_LAST=$ev python scripts/prof_run.py --lattice 400,400,40 --R 32,16,8 --M 20 --reps 2 2>&1 | sed "s/^/ev=$ev /"
KPM_V_EVICT_LAST=$ev python scripts/prof_run.py --lattice 200,100,40 --R 32,16,8 --M 20 --reps 2 2>&1 | sed "s/^/C3 ev=$ev /"
done
KPM_V_EVICT_LAST=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:aug_spmmv -s 1 -c 1 python scripts/prof_run.py --lattice 400,400,40 --R 32 --M 8 > gpurun_out/ncu_c4b.txt 2>&1
grep -E "dram__bytes|duration|hit_rate" gpurun_out/ncu_c4b.txt
