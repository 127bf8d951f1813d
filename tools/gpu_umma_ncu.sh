mkdir -p gpurun_out/umma
for c in grid rgg_spatial_ids; do
  for k in "k_tile_umma:umma:tile-umma" "k_tile_excl_bits:bits:tile"; do
    rx=$(echo $k | cut -d: -f1); nm=$(echo $k | cut -d: -f2); cand=$(echo $k | cut -d: -f3)
    CAND=$cand timeout 600 ncu --set full --clock-control none -k regex:"$rx" -s 0 -c 1 -o gpurun_out/umma/full_cand_${nm}_$c python tools/ncu_target.py $c > gpurun_out/umma/ncu_${nm}_$c.log 2>&1; echo ncu_${nm}_$c=$?
  done
done
