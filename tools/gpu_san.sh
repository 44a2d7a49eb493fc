#!/bin/bash
mkdir -p gpurun_out
for t in memcheck synccheck racecheck; do timeout 400 compute-sanitizer --tool $t python tools/sanitize_step.py > gpurun_out/san_$t.txt 2>&1; echo $t; tail -1 gpurun_out/san_$t.txt; done
