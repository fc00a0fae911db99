#!/bin/bash
# Standard GPU-box session: parity tests, smoke, benches (each under its own
# timeout), outputs under gpurun_out/<tag>_*.  Usage: tools/gpu_suite.sh TAG [WHAT...]
# WHAT: tests smoke bench bench4 bench5 bench3 bench1 launches ncu
set -u
tag=${1:-run}; shift || true
what=${*:-"tests smoke bench"}
mkdir -p gpurun_out
o=gpurun_out/${tag}
for w in $what; do
  case $w in
    tests)  timeout 900 python -m pytest tests -x -q -m gpu > ${o}_pytest.log 2>&1; echo "rc=$?" >> ${o}_pytest.log ;;
    smoke)  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1; echo "rc=$?" >> ${o}_smoke.log ;;
    bench)  timeout 900 python bench.py > ${o}_bench.json 2> ${o}_bench.err; echo "rc=$?" >> ${o}_bench.err ;;
    bench1) timeout 600 python bench.py --workload config1 --steps 50 > ${o}_bench1.json 2> ${o}_bench1.err; echo "rc=$?" >> ${o}_bench1.err ;;
    bench3) timeout 900 python bench.py --workload config3 > ${o}_bench3.json 2> ${o}_bench3.err; echo "rc=$?" >> ${o}_bench3.err ;;
    bench4) timeout 900 python bench.py --workload config4 --steps 20 > ${o}_bench4.json 2> ${o}_bench4.err; echo "rc=$?" >> ${o}_bench4.err ;;
    bench5) timeout 600 python bench.py --workload config5 --steps 20 > ${o}_bench5.json 2> ${o}_bench5.err; echo "rc=$?" >> ${o}_bench5.err ;;
    ref)    timeout 600 python bench.py --impl reference --steps 5 > ${o}_ref.json 2> ${o}_ref.err; echo "rc=$?" >> ${o}_ref.err ;;
    launches)
      cmd="python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
      timeout 600 $cmd > ${o}_plain.log 2>&1 && \
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
        --log-file ${o}_launches.csv $cmd > ${o}_ncu_launches.log 2>&1; echo "rc=$?" >> ${o}_ncu_launches.log ;;
    ncu)
      cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
      timeout 600 $cmd > ${o}_plain_full.log 2>&1 && \
      timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:ew_(step_|step16_)?kernel" -s 5 -c 5 \
        -o ${o}_prof_ew $cmd > ${o}_ncu_full.log 2>&1; echo "rc=$?" >> ${o}_ncu_full.log ;;
  esac
done
echo suite-done
