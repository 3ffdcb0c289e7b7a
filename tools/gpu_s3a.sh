mkdir -p gpurun_out
./tools/micro/dmma_lat > gpurun_out/s3_dmma_lat.txt 2>&1
bash tools/ab_pdl.sh > gpurun_out/s3_ab_pdl.txt 2>&1
TAG=s3a bash tools/gpu_check.sh
