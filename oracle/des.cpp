// des.cpp -- placeholder (DES oracle added later)
#include "oracle.h"
