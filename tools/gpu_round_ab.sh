set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge_cols.py -m gpu -x -q > gpurun_out/pytest_r2f.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2f.log
bash tools/ab_bench.sh r2f C4 "KDB_ROUND2=1" "KDB_ROUND2=0"
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
for S in 1 0; do
KDB_ROUND2=$S ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2f_$S.csv python bench.py $ARGS > /dev/null 2>&1; echo "ncu rc=$?"
python - $S <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/launches_r2f_{sys.argv[1]}.csv").readlines()[3:]))[1:]
for r in rows:
    if "light_round" in r[4]:
        print(r[0], r[4].split("(")[0][-30:], r[8], float(r[-1]) / 1e3, "us")
PY
done
bash tools/ab_bench.sh r2f3 C3 "KDB_ROUND2=1" "KDB_ROUND2=0"
bash tools/ab_bench.sh r2f2 C2 "KDB_ROUND2=1" "KDB_ROUND2=0"
