mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 1 --rows 1048576 > gpurun_out/s3s_gloo2.json 2> gpurun_out/s3s_gloo2.err; echo "gloo2 rc=$?"; tail -1 gpurun_out/s3s_gloo2.json | cut -c1-600
timeout 900 python bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/s3s_ref2.json 2> gpurun_out/s3s_ref2.err; echo "ref2 rc=$?"; tail -1 gpurun_out/s3s_ref2.json | cut -c1-300
tail -3 gpurun_out/s3s_gloo2.err
