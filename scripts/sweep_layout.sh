set -x
timeout 300 python scripts/sweep.py --parts 1536 --modes 5 --stages 2 --steps 100 2>&1 | grep part_nodes
timeout 300 python scripts/sweep.py --tuning first_touch=0 --parts 1536 --modes 5 --stages 2 --steps 100 2>&1 | grep part_nodes
timeout 300 python scripts/sweep.py --tuning hex_color=1 --parts 1536,2048 --modes 3,5,1 --stages 2 --steps 100 2>&1 | grep part_nodes
timeout 300 python scripts/sweep.py --config cfg3 --parts 1536 --modes 3 --stages 2 --steps 100 2>&1 | grep part_nodes
timeout 300 python scripts/sweep.py --tuning first_touch=0 --config cfg3 --parts 1536 --modes 3 --stages 2 --steps 100 2>&1 | grep part_nodes
