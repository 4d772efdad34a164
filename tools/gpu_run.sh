#!/bin/bash
# One gpurun session: build, smoke, GPU tests, bench, ncu launch list + full capture.
# usage: tools/gpu_run.sh TAG [stages...]   stages: smoke tests bench ncu_list ncu_full
TAG=${1:-r01}; shift
STAGES=${*:-"smoke tests bench ncu_list ncu_full"}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > "$OUT/nvsmi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo BUILD FAILED; tail -30 "$OUT/build.log"; exit 1; }
for st in $STAGES; do
  case $st in
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"; tail -3 "$OUT/smoke.log";;
    tests) timeout 1500 python -m pytest tests -q -m gpu -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?"; tail -15 "$OUT/pytest_gpu.log";;
    quicktests) timeout 900 python -m pytest tests -q -m gpu -x -k "not full_size" > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?"; tail -15 "$OUT/pytest_gpu.log";;
    bench) timeout 900 python bench.py --steps 10 --warmup 3 > "$OUT/bench_c5.log" 2>&1; echo "bench rc=$?"; tail -2 "$OUT/bench_c5.log";;
    bench_all)
      for c in c3 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/bench_$c.log" 2>&1; echo "bench $c rc=$?"; tail -1 "$OUT/bench_$c.log"; done
      for F in 16 32 64 128; do timeout 300 python bench.py --config c2 --F $F --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/bench_c2_F$F.log" 2>&1; tail -1 "$OUT/bench_c2_F$F.log"; done
      timeout 600 python bench.py --config c3 --partition warp --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/bench_c3_warp.log" 2>&1; tail -1 "$OUT/bench_c3_warp.log";;
    ab)  # A/B of kernel variants selected by environment (AB_VAR=values, e.g. AGCN_SPMM_U=4,8)
      for c in ${AB_CONFIGS:-c5 c4}; do for v in ${AB_VALUES//,/ }; do
        env ${AB_VAR}=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cusparse > "$OUT/ab_${c}_${AB_VAR}_$v.log" 2>&1
        echo "ab $c $AB_VAR=$v: $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'spmm', round(d['spmm_only']['ms_per_layer'],3), 'plan', round(d['plan_ms'],3))" "$OUT/ab_${c}_${AB_VAR}_$v.log" 2>&1 | tail -1)"
      done; done;;
    probe)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gather_probe.cu -o /tmp/gather_probe -lcuda > "$OUT/probe_build.log" 2>&1
      for a in "262144 67108864 0" "262144 67108864 1" "466000 67108864 1" "8388608 67108864 1" "8388608 67108864 0"; do
        timeout 300 /tmp/gather_probe $a >> "$OUT/probe.log" 2>&1; done; tail -60 "$OUT/probe.log";;
    l2probe)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/l2_probe.cu -o /tmp/l2_probe > "$OUT/l2probe_build.log" 2>&1
      for a in "8388608 67108864 390000 1.0" "8388608 67108864 390000 0.8" "466000 67108864 466000 0.5" "466000 67108864 300000 0.5"; do
        timeout 300 /tmp/l2_probe $a >> "$OUT/l2probe.log" 2>&1; done; cat "$OUT/l2probe.log";;
    ncu_list)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
        --log-file "$OUT/launches_c5.csv" python bench.py --profile --steps 2 --warmup 1 > "$OUT/ncu_list.log" 2>&1; echo "ncu_list rc=$?";;
    ncu_ab)  # full ncu capture of the SpMM kernel per config x variant (AB_VAR/AB_VALUES)
      for c in ${AB_CONFIGS:-c5 c4}; do for v in ${AB_VALUES//,/ }; do
        env ${AB_VAR}=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_ -s 3 -c 1 \
          -o "$OUT/prof_${c}_${AB_VAR}_$v" -f python bench.py --profile --config $c --steps 1 --warmup 1 > "$OUT/ncu_${c}_$v.log" 2>&1; echo "ncu $c $v rc=$?"
        python tools/ncu_summary.py "$OUT/sum_${c}_${AB_VAR}_$v" "$OUT/prof_${c}_${AB_VAR}_$v.ncu-rep" | tail -1
        python tools/ncu_stalls.py "$OUT/prof_${c}_${AB_VAR}_$v.ncu-rep" 30 > "$OUT/stalls_${c}_${AB_VAR}_$v.txt"
        [ -n "$KEEP_REP" ] || rm -f "$OUT/prof_${c}_${AB_VAR}_$v.ncu-rep"
      done; done;;
    ncu_full)
      for c in c5 c4 c3; do
        timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spmm_ -s 3 -c 1 \
          -o "$OUT/prof_$c" -f python bench.py --profile --config $c --steps 1 --warmup 1 > "$OUT/ncu_full_$c.log" 2>&1; echo "ncu_full $c rc=$?"
        python tools/ncu_summary.py "$OUT/sum_$c" "$OUT/prof_$c.ncu-rep" | tail -1
        python tools/ncu_stalls.py "$OUT/prof_$c.ncu-rep" 30 > "$OUT/stalls_$c.txt"
        [ -n "$KEEP_REP" ] || rm -f "$OUT/prof_$c.ncu-rep"
      done;;
  esac
done
ls -la "$OUT"
