#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench (C1 + C2), ncu launch list and
# full captures of the hot kernels.  Usage (under gpurun): bash tools/gpu_round.sh [tag]
set -x
TAG=${1:-r2}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --workload clf-c2 --no-micro > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-micro > $O/ncu_launch_bench.log 2>&1
python tools/launch_summary.py $O/launches.csv 30 > $O/launches_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c2.csv \
   python bench.py --workload clf-c2 --steps 1 --warmup 3 --no-cpu-baseline --no-micro > $O/ncu_launch_bench_c2.log 2>&1
python tools/launch_summary.py $O/launches_c2.csv 30 > $O/launches_c2_summary.txt 2>&1
timeout 600 env EAGER=1 REPS=2 ncu --set full --clock-control none --import-source on -k regex:"k_eprop_t|k_prep" -s 2 -c 2 \
   -o $O/eprop_c1 -f python tools/profile_eprop.py c1 > $O/ncu_eprop.log 2>&1
timeout 600 env EAGER=1 REPS=2 ncu --set full --clock-control none --import-source on -k regex:"k_eprop_t|k_prep" -s 2 -c 2 \
   -o $O/eprop_c2 -f python tools/profile_eprop.py c2 > $O/ncu_eprop_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_clf_fwd2|k_clf_readout" -s 50 -c 2 \
   -o $O/forward_c1 -f python tools/profile_forward.py c1 > $O/ncu_forward.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_clf_spikes|k_clf_xbar" -c 2 \
   -o $O/inputs_c1 -f python tools/profile_forward.py c1 > $O/ncu_inputs.log 2>&1
timeout 900 env ROWS=262144 ncu --set full --clock-control none --import-source on \
   -k regex:"k_deepr_elim|k_deepr_form_rows" -c 6 -o $O/deepr -f python tools/mupdate_breakdown.py > $O/ncu_deepr.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_prop_bucketed|k_prop_atomic" -c 4 \
   -o $O/prop -f python tools/profile_prop.py > $O/ncu_prop.log 2>&1
ls -la $O
