#!/bin/bash
timeout 120 python tools/time_groups.py rot 1 2>&1
timeout 120 python tools/time_groups.py norot 1 2>&1
