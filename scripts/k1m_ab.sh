#!/bin/bash
# K1m vs K1 (butterfly) and K1m work-split configs, flushed-L2 event timing.
python scripts/k1_ab.py 'MRFP4_K1_MMA=0' 'MRFP4_K1M_CFG=0' 'MRFP4_K1M_CFG=1' 'MRFP4_K1M_CFG=2' 'MRFP4_K1M_CFG=3'
