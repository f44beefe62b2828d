// TEST INFRASTRUCTURE: the reference header <rx/parallel.hpp> resolves to the B200 facade.
#pragma once
#include "rx_b200.hpp"
