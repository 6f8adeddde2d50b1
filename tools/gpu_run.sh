#!/usr/bin/env bash
# One parameterised GPU-box runner (replaces the round-1 one-off session scripts).
# Run through gpurun from the repo root:
#   gpurun --timeout S -- 'bash tools/gpu_run.sh <task> [args]'
# Tasks (each writes its logs under gpurun_out/):
#   smoke                     __graft_entry__.smoke()
#   tests [pytest -k expr]    pytest -m gpu (optionally filtered)
#   bench [bench.py args]     one bench line  -> gpurun_out/bench_<tag>.jsonl (tag = $TAG or "run")
#   ref [bench.py args]       the reference arm (bench.py --impl reference)
#   launches [bench.py args]  ncu launch list (gpu__time_duration.sum, cold) of a short bench run;
#                             NCU_EXTRA_METRICS=dram__bytes_read.sum,dram__bytes_write.sum adds DRAM bytes per kernel
#   ncu <kernel-regex> <count> [bench.py args]   ncu --set full of one kernel from a short bench run
#   py <script> [args]        any python tool (tools/*.py)
set -u
mkdir -p gpurun_out
task=${1:-smoke}; shift || true
tag=${TAG:-run}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
case "$task" in
  smoke) python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log ;;
  tests)
    if [ $# -gt 0 ]; then timeout ${PYTEST_TIMEOUT:-2400} python -m pytest tests -q -m gpu --timeout=${TEST_TIMEOUT:-900} -k "$*" > gpurun_out/pytest_$tag.log 2>&1
    else timeout ${PYTEST_TIMEOUT:-2400} python -m pytest tests -q -m gpu --timeout=${TEST_TIMEOUT:-900} > gpurun_out/pytest_$tag.log 2>&1; fi
    echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/pytest_$tag.log | tail -15 ;;
  bench) timeout ${BENCH_TIMEOUT:-2400} python bench.py "$@" > gpurun_out/bench_$tag.jsonl 2> gpurun_out/bench_$tag.err
    echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$tag.jsonl; tail -5 gpurun_out/bench_$tag.err ;;
  ref) timeout ${BENCH_TIMEOUT:-2400} python bench.py --impl reference "$@" > gpurun_out/ref_$tag.jsonl 2> gpurun_out/ref_$tag.err
    echo "ref rc=$?"; tail -c 2000 gpurun_out/ref_$tag.jsonl; tail -5 gpurun_out/ref_$tag.err ;;
  launches) timeout ${BENCH_TIMEOUT:-2400} ncu --metrics gpu__time_duration.sum${NCU_EXTRA_METRICS:+,$NCU_EXTRA_METRICS} --clock-control none -c ${NCU_COUNT:-2000} --csv \
      --log-file gpurun_out/launches_$tag.csv python bench.py --no-cpu-baseline "$@" > gpurun_out/launches_$tag.log 2>&1
    echo "launches rc=$?"; python tools/ncu_summary.py launches gpurun_out/launches_$tag.csv gpurun_out/launches_$tag.json | tail -20 ;;
  ncu) k=$1; c=$2; shift 2
    timeout ${BENCH_TIMEOUT:-2400} ncu --set full --import-source on --clock-control none -k "regex:$k" -c "$c" \
      -o gpurun_out/ncu_$tag python bench.py --no-cpu-baseline "$@" > gpurun_out/ncu_$tag.log 2>&1
    echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$tag.log ;;
  py) s=$1; shift; timeout ${PY_TIMEOUT:-2400} python "$s" "$@" > gpurun_out/py_$tag.log 2>&1; echo "py rc=$?"; tail -40 gpurun_out/py_$tag.log ;;
  *) echo "unknown task $task"; exit 2 ;;
esac
