#!/bin/bash
python -m pytest tests -m gpu -q -k "stream_frame_queue or c4_long" 2>&1 | tail -3
python scripts/c4_es_speed.py 65536 1.1 2>&1 | tail -6
