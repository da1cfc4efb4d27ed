# synccheck of the folded-LayerNorm layer: repeat, unfolded, PDL off
python __graft_entry__.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/sanitizer
run() { timeout 900 compute-sanitizer --tool synccheck --print-limit 4 python scripts/sanitize.py $@ > gpurun_out/sanitizer/sc_$1_$2_$OPARA_PDL.txt 2>&1; echo "$@ pdl=$OPARA_PDL rc=$? $(grep -E 'ERROR SUMMARY|ok=|Barrier error|block \(' gpurun_out/sanitizer/sc_$1_$2_$OPARA_PDL.txt | sort | uniq -c | head -6 | tr '\n' ' ')"; }
export OPARA_PDL=1; run bert_fold fold; run bert_fold fold; run bert_fold nofold; run bert_layer fold
export OPARA_PDL=0; run bert_fold fold
