# ncu --set full of one r=1 B=128 FP32 conv launch (128x64 GEMM kernel for every layer)
NCU=/usr/local/cuda/bin/ncu
SLIM_F32_GEMM128=1 $NCU --set full --clock-control none --import-source on -k "regex:conv_f32_gemm_kernel" -s 390 -c 1 -o /tmp/f32_r1 \
    python tools/layer_times.py 128 3 bn fp32 > /dev/null 2>&1
$NCU -i /tmp/f32_r1.ncu-rep --page details --csv > gpurun_out/r02_ncu_f32_r1.csv
$NCU -i /tmp/f32_r1.ncu-rep --page raw --csv > gpurun_out/r02_ncu_f32_r1_raw.csv
