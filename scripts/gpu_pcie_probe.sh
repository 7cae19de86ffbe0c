LPQ_STREAM_TRACE=1 timeout 600 python scripts/pcie_e2e_probe.py 2>&1 | grep "e2e\|stream" | tail -4
