nvidia-smi topo -m 2>&1 | head -20
echo "--- nodes"; ls /sys/devices/system/node/ 2>&1; for n in /sys/devices/system/node/node*; do echo $n $(cat $n/cpulist) $(grep MemTotal $n/meminfo); done
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1)
echo "bus $BUS"; B=$(echo $BUS | tr 'A-F' 'a-f' | sed 's/^0000//'); ls /sys/bus/pci/devices/ | grep -i "${B#0000}" ; for d in /sys/bus/pci/devices/*${B:4}; do echo $d numa=$(cat $d/numa_node) ; cat $d/current_link_speed $d/current_link_width 2>/dev/null; done
echo "--- affinity"; python -c "import os; print(sorted(os.sched_getaffinity(0)))"; nproc; lscpu | head -30; which numactl taskset
python tools/pcie.py 2>&1 | head -20
