# Figs. 8-9 analysis kernels: parity tests, device timing, then one ncu metrics pass.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_analysis.log 2>&1 || { tail -30 gpurun_out/pytest_analysis.log; exit 1; }
tail -2 gpurun_out/pytest_analysis.log
python scripts/fig9_kernels.py --out gpurun_out/fig9_time.json > gpurun_out/fig9_time.log 2>&1 || { tail -20 gpurun_out/fig9_time.log; exit 1; }
cat gpurun_out/fig9_time.log
python scripts/fig9_kernels.py --ncu > gpurun_out/fig9_ncu_plain.log 2>&1 || { tail -20 gpurun_out/fig9_ncu_plain.log; exit 1; }
M=$(cd scripts && python -c "import fig9_kernels as f; print(','.join(f.METRICS))")
ncu --metrics $M --clock-control none -k regex:aug_spmmv_tiled --csv --log-file gpurun_out/fig9_ncu.csv \
    python scripts/fig9_kernels.py --ncu > gpurun_out/fig9_ncu.log 2>&1
echo ncu=$?
