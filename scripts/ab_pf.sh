#!/bin/bash
# A/B the L2 prefetch distance of the swap-mode GEMMs in one box session
for cfg in "0 0" "4 0" "8 0" "8 1" "16 0" "0 0"; do
  set -- $cfg
  echo "== TAMOE_PF_DIST=$1 TAMOE_PF_B=$2"
  TAMOE_PF_DIST=$1 TAMOE_PF_B=$2 python scripts/gemm_micro.py 2>&1 | grep -E "C2 fwd|C2 dgrad|ep8 fwd|dense 16384" | cut -c1-120
done
