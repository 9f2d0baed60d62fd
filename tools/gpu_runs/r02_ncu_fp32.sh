# ncu --set full of the FP32-mode conv kernels (r=1, B=128 chain: one launch of each GEMM variant)
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k "regex:conv_f32_gemm" -s 2 -c 1 -o /tmp/f32_256 \
    python tools/layer_times.py 128 1 bn fp32 > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k "regex:conv_f32_gemm_kernel" -s 20 -c 1 -o /tmp/f32_128 \
    python tools/layer_times.py 128 1 bn fp32 > /dev/null 2>&1
for f in f32_256 f32_128; do $NCU -i /tmp/$f.ncu-rep --page details --csv > gpurun_out/r02_ncu_$f.csv; $NCU -i /tmp/$f.ncu-rep --page raw --csv > gpurun_out/r02_ncu_${f}_raw.csv; done
ls -la gpurun_out/
