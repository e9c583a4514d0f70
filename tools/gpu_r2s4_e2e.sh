# e2e repeatability: HostPipeline repeats (chunk x depth), raw PCIe bandwidth
timeout 120 python tools/pcie_bw.py 2>&1 | tail -8
for c in 4 8; do for dp in 2 3; do timeout 300 python tools/e2e_probe.py $c inplace $dp 2>&1 | tail -6; done; done
