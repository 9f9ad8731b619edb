#!/bin/bash
# One GPU round trip: parity tests, smoke, bench line, ncu launch list and a
# full ncu capture of the dominant kernel.  Outputs land in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2001_04206_b200._build >/dev/null 2>&1
TAG=${TAG:-r1}
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests -q -m gpu -p no:hypothesispytest > gpurun_out/pytest_gpu_$TAG.txt 2>&1
  tail -3 gpurun_out/pytest_gpu_$TAG.txt
  timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
fi
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.json
if [ "${NCU:-1}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu ${BENCH_ARGS:-} > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_sgd_cluster} -s 1 -c 1 \
      -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu --epoch 4000 ${BENCH_ARGS:-} > /dev/null 2>&1
  ls -la gpurun_out/ | grep $TAG
fi
