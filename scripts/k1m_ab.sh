#!/bin/bash
# K1m work-split configs vs the butterfly kernel, flushed-L2 event timing.
python scripts/k1_ab.py 'MRFP4_K1_MMA=0' 'MRFP4_K1M_CFG=0' 'MRFP4_K1M_CFG=1'
