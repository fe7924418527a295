#!/bin/bash
# A/B of densify shapes (RFL_DENSIFY="v<6|9>:256:<tile KB>:<8|16>:<2|3|4>") on the kbench densify cases.
C=${CASES:-densify_cfg1,densify_bf16_cfg1,densify_norm_cfg2}
for V in ${VARIANTS:-v9:256:80:16:2 v9:256:40:8:3 v9:256:40:8:4 v6:256:80:16:2 v6:256:40:8:3}; do
  echo "## $V"
  RFL_DENSIFY=$V timeout 300 python scripts/kbench.py --cases $C --steps 20 2>/dev/null
done
