#!/bin/bash
# Build libdsv locally, then run a command on a B200 through gpurun.
# usage: tools/gpu.sh [--timeout S] [--gpus N] '<command>'
set -e
cd /root/repo
python paper_2502_07590_b200/build.py > /dev/null
TO=600; GP=1
while [[ "$1" == --* ]]; do
  case "$1" in
    --timeout) TO=$2; shift 2;;
    --gpus) GP=$2; shift 2;;
  esac
done
exec timeout $((TO + 1800)) /usr/local/graft/bin/gpurun --timeout "$TO" --gpus "$GP" -- "export DSV_NO_BUILD=1; $1"
