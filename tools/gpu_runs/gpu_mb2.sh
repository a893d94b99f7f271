timeout 60 ./tools/desc_shift_test > gpurun_out/desc_shift2.json 2>&1; cat gpurun_out/desc_shift2.json
