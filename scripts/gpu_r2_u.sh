# per-phase stamps of BERT's GEMMs (folded LayerNorm) in the sequential graph
export OPARA_NVCC_FLAGS=-DOPARA_PHASE_PROBE
python -m paper_2312_10351_b200.build > /dev/null 2>&1 || exit 1
timeout 900 python scripts/phase_probe.py bert_base bf16 --grids bounded --slot sequential --splitk auto 2>&1 | grep -v Warn | tail -12
unset OPARA_NVCC_FLAGS
python -m paper_2312_10351_b200.build > /dev/null 2>&1
