#!/bin/bash
# One GPU round trip for the round's evidence: the GPU parity suite, smoke,
# the bench lines (default C5 + C3 + C2), the ncu launch list of the default
# bench command, one full ncu capture of its dominant kernel, and the DRAM
# traffic per launch (profiles/traffic.json).  Outputs: gpurun_out/${TAG}_*.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2}
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -q -m gpu -p no:hypothesispytest > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
  tail -3 gpurun_out/${TAG}_pytest_gpu.txt
  timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.txt 2>&1; tail -1 gpurun_out/${TAG}_smoke.txt
fi
for w in ${WORKLOADS:-c5 c3 c2}; do
  timeout 900 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
  tail -c 300 gpurun_out/${TAG}_bench_$w.json; echo
done
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_gemm_h3} -s 3 -c 1 \
      -o gpurun_out/${TAG}_full_c5 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
  timeout 1500 python tools/ncu_traffic.py > gpurun_out/${TAG}_traffic.txt 2>&1
  ls -la gpurun_out/ | grep ${TAG}_
fi
