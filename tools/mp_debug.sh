#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python tools/mp_debug2.py pcgxdbg3 2 0 > gpurun_out/mpd3_r0.log 2>&1 &
python tools/mp_debug2.py pcgxdbg3 2 1 > gpurun_out/mpd3_r1.log 2>&1
wait
echo done
