cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=r02s
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 1500 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | tail -8
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout -s KILL 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo -n "bench rc=$? "; python scripts/show.py gpurun_out/${TAG}_bench.json
