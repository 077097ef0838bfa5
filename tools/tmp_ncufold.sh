mkdir -p gpurun_out
bash tools/ncu_kernel.sh k_gemm_fold c5 nf_c5 WINO_FOLD=2
bash tools/ncu_kernel.sh k_gemm_fold c3 nf_c3 WINO_FOLD=1
bash tools/ncu_kernel.sh k_gemm c5 nu_c5 WINO_FOLD=0
python tools/ncu_summary.py gpurun_out/nf_c5_raw.csv gpurun_out/nf_c3_raw.csv gpurun_out/nu_c5_raw.csv
