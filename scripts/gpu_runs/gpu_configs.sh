# other bench configurations after the diagonal-first order (C2, C4 at N=1) + the reference arm
mkdir -p gpurun_out
for c in C2 C4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-r-sweep --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"; cut -c1-220 gpurun_out/cfg_$c.json; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/ref.json
