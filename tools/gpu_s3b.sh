mkdir -p gpurun_out
bash tools/ab_libs2.sh build/ab/libCPF.so build/ab/libBASE.so build/ab/libCPF2.so > gpurun_out/s3_ab_cpf.txt 2>&1
