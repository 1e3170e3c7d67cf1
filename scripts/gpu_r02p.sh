mkdir -p gpurun_out
cd scripts && timeout 120 ./drain_rate > ../gpurun_out/r02p.txt 2>&1; cd ..
cat gpurun_out/r02p.txt
