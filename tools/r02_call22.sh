# round 2, call 22: the lazy-bound debug build (every Montgomery product traps unless its raw output < 2N) over
# every kernel path of the final tree (n0' slot, L = 6 square unroll 16), with its negative control —
# the bounds checks of our own that stand in for compute-sanitizer, which this pool has closed
set -x
TAG=r02v
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python tools/debug_bounds.py > $OUT/${TAG}_debug_bounds.json 2> $OUT/${TAG}_debug_bounds.err
tail -c 600 $OUT/${TAG}_debug_bounds.json
