#!/bin/bash
# Round-2 pass S: host page size of the pinned pool vs PCIe copy rates.
timeout 300 python tools/pcie_hugepage_probe.py 2>&1 | tail -3
timeout 300 python tools/pcie_hugepage_probe.py 2>&1 | tail -1
