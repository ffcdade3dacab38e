#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu -rs -k "not fullsize" > gpurun_out/p9_gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/p9_gputests.log
python tools/sanitize_run.py > gpurun_out/p9_san_plain.log 2>&1
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/p9_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/p9_san_$tool.log
done
echo done
