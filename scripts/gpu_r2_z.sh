# round-2 closing evidence: GPU tests, smoke, every config's bench line, reference arm, ncu (Inception-v3 fp32, BERT)
bash scripts/gpu_r2_final.sh
NCU_SPECS="inception_v3 f32 conv2d_tc_tf32x3|bert_base bf16 conv2d_tc_bf16" bash scripts/gpu_ncu_r02.sh 2>&1 | tail -12
