#!/bin/bash
# config-3 (B=1) step time with the attention variant chosen by attn_split vs forced cluster split
timeout 600 python bench.py --config 3 --steps 64 --warmup 8 2>&1 | tail -1 | cut -c1-1200
