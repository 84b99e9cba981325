# one GPU session: c5 headline bench (N=1), the N=2 sharded path on one shared device,
# the reference arm, and the c5 launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -z "$NO_N2" ]; then
PHMM_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench_n2 rc=$?
cat gpurun_out/bench_n2.json; tail -5 gpurun_out/bench_n2.err
fi
if [ -z "$NO_REF" ]; then
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
fi
for W in ${PROFILE_WORKLOADS:-}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_${W}.csv python tools/profile_run.py $W 2 --retry > gpurun_out/launches_${W}.log 2>&1
  echo launches $W rc=$?
done
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
ls gpurun_out
