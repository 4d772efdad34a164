# One gpurun session that produces the evidence of a round: build, smoke, GPU tests, the default
# bench line, the kernel launch list of the default bench (ncu, cold per kernel), ncu --set full
# summaries of the SpMM kernels on C5 / C4 / C3 (reports deleted after summarising: gpurun_out
# must stay < 64 MiB).   usage: bash tools/final_run.sh TAG [stages]
TAG=${1:-final}; shift
STAGES=${*:-"smoke tests bench launches ncu"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
for st in $STAGES; do case $st in
  smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log;;
  tests) timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log;;
  bench) timeout 1500 python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?"; tail -1 $OUT/bench.log > $OUT/bench_line.json;;
  launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python bench.py --profile --steps 2 --warmup 1 > $OUT/launches.log 2>&1; echo "launches rc=$?"; python tools/launches.py $OUT/launches_c5.csv > $OUT/launches_c5.txt 2>&1; head -14 $OUT/launches_c5.txt;;
  ncu) for c in c5 c4 c3; do
         timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_wide|k_spmm_chunks" -s $([ $c = c3 ] && echo 2 || echo 4) -c 2 -o $OUT/prof_$c -f python bench.py --profile --config $c --steps 1 --warmup 3 > $OUT/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
         python tools/ncu_stalls.py $OUT/prof_$c.ncu-rep 25 > $OUT/stalls_$c.txt 2>&1
       done
       python tools/ncu_summary.py $OUT/ncu_sum $OUT/prof_c5.ncu-rep $OUT/prof_c4.ncu-rep $OUT/prof_c3.ncu-rep | tail -8
       rm -f $OUT/*.ncu-rep;;
esac; done
ls -la $OUT
