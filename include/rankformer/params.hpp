// SPDX-License-Identifier: Apache-2.0
// Drop-in include path: a caller written against the reference's rankformer/params.hpp compiles
// unchanged with -I<repo>/include; every hot-path declaration lives in reference_api.hpp.
#pragma once
#include "reference_api.hpp"
