bash tools/profile.sh > gpurun_out/g12_profile.log 2>&1; echo profile $?
ls gpurun_out/*.ncu-rep gpurun_out/launches.csv
