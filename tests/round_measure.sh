# Round-end measurement (GPU): the GPU test suite, smoke, the bench lines (GAN trained / He-init, spline,
# reference arm), the ncu launch lists of both bench modes and one --set full capture of the generator.
set -x
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q > gpurun_out/final/gputests.log 2>&1; echo rc=$? >> gpurun_out/final/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
python bench.py > gpurun_out/final/bench_gan.json 2> gpurun_out/final/bench_gan.err
python bench.py --mode spline > gpurun_out/final/bench_spline.json 2> gpurun_out/final/bench_spline.err
python bench.py --weights he --no-cpu-baseline > gpurun_out/final/bench_he.json 2> gpurun_out/final/bench_he.err
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_gan.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu_gan.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_spline.csv python bench.py --mode spline --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu_spline.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gen_tc -s 1 -c 1 -o gpurun_out/final/gen_full python tests/tc_profile.py 2048 2 > gpurun_out/final/ncu_gen_full.log 2>&1
ls -la gpurun_out/final
