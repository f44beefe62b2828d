// TEST INFRASTRUCTURE: the reference header <rx/regex.hpp> resolves to the B200 facade.
#pragma once
#include "rx_b200.hpp"
