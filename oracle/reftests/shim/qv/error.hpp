// qv/error.hpp -> the qv:: drop-in (test infrastructure: lets the reference's
// own test files compile unchanged against paper_2305_10863_b200/cpp).
#pragma once
#include "qv_b200.hpp"
