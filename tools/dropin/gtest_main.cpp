#include "gtest/gtest.h"
int main() { return ::testing::RunAll(); }
