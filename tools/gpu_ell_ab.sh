# same-box A/B of the light ELL layout: row-major (libkdb.so) vs planes (libkdb_ellplanes.so), alternating
mkdir -p gpurun_out
TAG=${1:-ell}
for rep in 1 2; do for lib in libkdb.so libkdb_ellplanes.so; do
KDB_LIBRARY=$PWD/paper_2009_04552_b200/lib/$lib timeout 900 python bench.py --order ${ORDER:-inertial} --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/bench_${TAG}_$lib.jsonl > gpurun_out/bench_${TAG}_${lib}_$rep.log 2>&1; echo "$lib rep=$rep rc=$?"
done; done
