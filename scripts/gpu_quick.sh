#!/usr/bin/env bash
timeout 300 python scripts/dev_shared.py 2>&1 | tail -20
