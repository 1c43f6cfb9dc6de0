#!/bin/bash
# libdpp with device-side invariant checks (-DDPP_CHECKED) into ab_libs/checked.so
exec "$(dirname "$0")/variant_build.sh" checked "-DDPP_CHECKED"
