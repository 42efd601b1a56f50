bash abtest/run2.sh; bash abtest/run2.sh
