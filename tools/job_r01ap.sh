#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "
from paper_2411_18424_b200.dataplane import host_link_info
print(host_link_info('cuda:0'))"
nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.gen.gpumax,pcie.link.width.current,pcie.link.width.max --format=csv
