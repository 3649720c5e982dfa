#!/bin/bash
# Quick GPU check: selected tests (args = pytest -k expression / files), then the full suite.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${TAG:-q}
timeout -s KILL 600 python -m pytest "$@" -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/${TAG}_sel.log 2>&1
echo "selected rc=$?"; tail -30 gpurun_out/${TAG}_sel.log | grep -vE "^\s*$" | tail -25
