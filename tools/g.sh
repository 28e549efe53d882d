#!/bin/bash
# usage: tools/g.sh <logname> <timeout-s> '<command run on the GPU box from the repo root>'
cd /root/repo || exit 1
name=$1; to=$2; shift 2
/usr/local/graft/bin/gpurun --timeout "$to" -- "$@" > "gpurun_out/$name.log" 2>&1
echo "exit=$?"; grep -vE "^\[gpurun\] (send|merged)" "gpurun_out/$name.log" | tail -${TAILN:-12} | cut -c1-260
