# Full round evidence on one GPU (gpurun): GPU tests, tools/evidence.sh, the M10/M50/M200 lines,
# a 2-rank torchrun harness run and smoke(); then `python tools/evidence.py $TAG` here.
# usage: TAG=r02e bash tools/round_evidence_all.sh
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_${TAG:-r02}.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_${TAG:-r02}.log
bash tools/evidence.sh ${TAG:-r02}
for w in m10 m50 m200; do S=5; [ $w == m10 ] && S=400; timeout 900 python bench.py --workload $w --steps $S --warmup 3 --no-cpu-baseline > gpurun_out/bench_${w}_${TAG:-r02}.json 2> gpurun_out/bench_${w}_${TAG:-r02}.err; echo "$w rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --workload m10 > gpurun_out/bench_m10_2ranks_${TAG:-r02}.json 2> gpurun_out/bench_m10_2ranks_${TAG:-r02}.err; echo "2rank rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG:-r02}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG:-r02}.log
