# quick GPU check of selected tests: bash scripts/gpu/r2_quick.sh "<pytest -k expr>"
mkdir -p gpurun_out/quick
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/quick/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests -m gpu -q -k "$1" > gpurun_out/quick/pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/quick/pytest.log
