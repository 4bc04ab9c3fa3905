mkdir -p gpurun_out
V=paper_1712_02248_b200/build_var/drain1/libcnmf_b200.so
CNMF_XS=tf32 timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_i_tf32.txt 2>&1; grep "final\|relF" gpurun_out/c3_i_tf32.txt
CNMF_RECON=simt CNMF_XS=tf32 timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_i_tf32_rsimt.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_i_tf32_rsimt.txt | tr '\n' ' '; echo; grep "final" gpurun_out/c3_i_tf32_rsimt.txt
CNMF_LIB=$V CNMF_RECON=simt CNMF_XS=f16 timeout 600 python tools/c3_gpu_variants.py c3 > gpurun_out/c3_i_d1f16_rsimt.txt 2>&1; awk '{print $2, $8}' gpurun_out/c3_i_d1f16_rsimt.txt | tr '\n' ' '; echo; grep "final" gpurun_out/c3_i_d1f16_rsimt.txt
