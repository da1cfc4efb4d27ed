B=./scripts/micro/launch_overhead
for c in 25 98 148; do
$B empty $c; $B smem $c 0; $B smem $c 48; $B smem $c 100; $B smem $c 148; $B smem $c 200
$B tmem $c 16; $B tmem $c 148; $B tmem $c 148 2
done
