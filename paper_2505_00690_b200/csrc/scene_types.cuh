// Host<->device structs come from the public C ABI header (single source of truth).
#pragma once
#include "citywalk_b200.h"
