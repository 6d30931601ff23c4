# Regenerate the round's evidence on one GPU (outputs in gpurun_out/):
#   bench_n1.log            full default bench line (N = 1)
#   launches.csv            ncu launch list (gpu__time_duration) of the act bench
#   q.ncu-rep / dq.ncu-rep  ncu --set full of one C2 quant (b=6) / dequant (b=5) launch
#   acc.ncu-rep             ncu --set full of one K3 launch (2^28 params, fp32 local)
set -x
python bench.py > gpurun_out/bench_n1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_quant_warp<\(int\)6' -c 1 -o gpurun_out/q \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline > gpurun_out/ncu_q.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_dequant_warp<\(int\)5' -c 1 -o gpurun_out/dq \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline > gpurun_out/ncu_dq.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_accumulate_warp -c 1 -o gpurun_out/acc \
  python tools/microbench.py --which acc > gpurun_out/ncu_acc.log 2>&1
ls -la gpurun_out/
