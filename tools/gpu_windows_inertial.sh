# full-size window parity of the benchmarked path in the inertial order: C4 and C5/4,
# goldens from oracle/ runs; then ncu of the round-2 light round in that order
mkdir -p gpurun_out
timeout 1800 python tools/window_parity.py --config C4 --order inertial --workers 5 --out gpurun_out/window_parity_C4i.json --golden tests/golden/window_oracle_C4i.json > gpurun_out/windows_C4i.log 2>&1; echo "C4i rc=$?"
mkdir -p gpurun_out/golden; cp tests/golden/window_oracle_C4i.json gpurun_out/golden/ 2>/dev/null
timeout 1800 python tools/window_parity.py --config C5 --scale 0.25 --order inertial --workers 5 --out gpurun_out/window_parity_C5qi.json --golden tests/golden/window_oracle_C5qi.json > gpurun_out/windows_C5qi.log 2>&1; echo "C5qi rc=$?"
cp tests/golden/window_oracle_C5qi.json gpurun_out/golden/ 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_light_round -c 1 -o gpurun_out/lr_inertial_ncu python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 1 --warmup 0 > gpurun_out/lr_ncu.log 2>&1; echo "ncu rc=$?"
