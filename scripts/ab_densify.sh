#!/bin/bash
# A/B of densify variants (RFL_DENSIFY) on the kbench densify cases.
C=${CASES:-densify_cfg1,densify_bf16_cfg1,densify_norm_cfg2}
for V in ${VARIANTS:-v2:512:100 v2:512:40 v2:256:80 v2:256:40 v2:256:20 v2:128:20 v3}; do
  echo "## $V"
  RFL_DENSIFY=$V timeout 300 python scripts/kbench.py --cases $C --steps 20 2>/dev/null
done
