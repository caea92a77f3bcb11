# Host facts that might separate the pool's two kinds of GPU box (tools only), then which
# D2H ring geometry this box's context picks.
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag 2>/dev/null
cat /proc/sys/kernel/numa_balancing 2>/dev/null | sed 's/^/numa_balancing /'
grep -m1 -o "iommu=[a-z]*\|intel_iommu=[a-z]*" /proc/cmdline 2>/dev/null; cat /proc/cmdline | cut -c1-200
lscpu | grep -E "MHz|Model:|Stepping|Flags" | cut -c1-120
nvidia-smi --query-gpu=name,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,driver_version --format=csv,noheader
nvidia-smi topo -m 2>/dev/null | head -4
grep -E "MemTotal|Hugepagesize|AnonHugePages" /proc/meminfo
bash tools/tune_check.sh 2>&1 | grep -E "D2H ring|e2e" | head -3
