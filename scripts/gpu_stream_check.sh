#!/bin/bash
python scripts/c4_es_speed.py 65536 1.1 2>&1 | tail -6
python scripts/c4_es_speed.py 65536 1.3 2>&1 | tail -6
