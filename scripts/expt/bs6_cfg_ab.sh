#!/bin/bash
# A/B of the super-block kernel's shape at low order (SB200_BS6_CFG, read per call)
for cfg in ${CFGLIST:-default lanes,0,12 lanes,0,14 lanes,0,16}; do
  if [ "$cfg" = default ]; then unset SB200_BS6_CFG; else export SB200_BS6_CFG=$cfg; fi
  SB200_BS6_TILED=0 timeout 300 python scripts/expt/time_bs6.py ${ORDERS:-2 3}
done
