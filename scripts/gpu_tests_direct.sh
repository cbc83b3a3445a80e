#!/bin/bash
python -m pytest tests -m gpu -q --durations=5 -k "direct or tuning or cpp or sweep or multi or per_frame or pins" 2>&1 | tail -25
