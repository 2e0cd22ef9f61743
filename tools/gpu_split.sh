#!/bin/bash
# On the GPU box: whole counts and 8-part splits (part by part, one GPU) of C4 / C5 / C3, total and per-vertex.
p() { python tools/phase_probe.py "$@" 2>&1 | grep -E "^[0-9]|part |parts=" | tail -10; }
echo "== C4 pv";  p --pv 1 --iters 2; p --pv 1 --iters 2 --parts 8
echo "== C4 total"; p --pv 0 --iters 2; p --pv 0 --iters 2 --parts 8
echo "== C5 total"; p --scale 26 --param 32 --pv 0 --iters 2; p --scale 26 --param 32 --pv 0 --iters 2 --parts 8
echo "== C5 pv"; p --scale 26 --param 32 --pv 1 --iters 2; p --scale 26 --param 32 --pv 1 --iters 2 --parts 8
echo "== C3 total"; p --kind kron --scale 22 --pv 0 --iters 2; p --kind kron --scale 22 --pv 0 --iters 2 --parts 8
