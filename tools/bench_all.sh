# Every bench line of the round (one JSON line per workload) into gpurun_out/<tag>_*.json.
# usage: bash tools/bench_all.sh <tag> [extra bench.py args]
T=${1:-r02}; shift
set -x
python bench.py "$@" > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.json 2>&1
for w in mixed drop drop-fwd ee vf demo; do
  python bench.py --workload $w --steps 20 --warmup 3 "$@" > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
python bench.py --eps 0.2 --steps 50 --warmup 3 --no-extras "$@" > gpurun_out/${T}_bench_eps0.2.json 2> gpurun_out/${T}_bench_eps0.2.err
python bench.py --eps 0.3 --steps 20 --warmup 3 --no-extras "$@" > gpurun_out/${T}_bench_eps0.3.json 2> gpurun_out/${T}_bench_eps0.3.err
python bench.py --n-total 1048576 --steps 20 --warmup 3 --no-extras --no-cpu-baseline "$@" > gpurun_out/${T}_bench_1m.json 2> gpurun_out/${T}_bench_1m.err
echo done
