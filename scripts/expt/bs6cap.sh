set -e
for lib in default c512t256 c1024t256 c1024t128; do
  if [ $lib = default ]; then L=""; else L="$PWD/scripts/expt/_bs6r/lib_$lib.so"; fi
  for cfg in "" "pairs,1,6" "pairs,1,8" "lanes,0,6" "lanes,0,8" "lanes,0,10"; do
    if [ -z "$cfg" ]; then
      SB200_LIB=$L timeout 300 python scripts/expt/time_bs6.py 1 2 3 7 | sed "s/^/$lib auto /"
    else
      SB200_LIB=$L SB200_BS6_CFG=$cfg timeout 300 python scripts/expt/time_bs6.py 1 2 3 7 | sed "s/^/$lib $cfg /"
    fi
  done
done
