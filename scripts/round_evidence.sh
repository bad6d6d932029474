#!/bin/bash
# One GPU call's worth of round-end evidence (run under gpurun):
#   pytest -m gpu, smoke(), the driver's bench command (ours + reference arm),
#   the ncu launch list of a short bench run.  Outputs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/ev_pytest.log 2>&1; tail -3 gpurun_out/ev_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; tail -2 gpurun_out/ev_smoke.log
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.log
tail -c 600 gpurun_out/ev_bench_ref.json
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.log
tail -c 300 gpurun_out/ev_bench.json; grep "\[bench\]" gpurun_out/ev_bench.log | tail -4
if [ "${EV_NCU:-1}" = "1" ]; then
  # only the timed swapped steps are profiled (bench.py: LMS_NCU_TIMED)
  LMS_NCU_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
      --log-file gpurun_out/ev_launches.csv \
      python bench.py --steps 2 --warmup 3 --tune-windows 0 --same-batch 0 --cpu-baseline 0 > gpurun_out/ev_ncu_bench.log 2>&1
  ls -la gpurun_out/ev_launches.csv
fi
