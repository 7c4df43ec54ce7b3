import sys, os
sys.path.insert(0, '/root/repo')
from tools.profile_one import coll
from paper_2511_04853_b200 import convert as cv, layouts as ly, sensor
n = 64*436*436
a, p = coll(sensor.SENSOR_SCHEMA, ly.AOS, n), coll(sensor.SENSOR_SCHEMA, ly.PER_FIELD, n)
print("a2p", cv.plan_info(cv.plan_desc(p.layout, a.layout, n), 0))
print("p2a", cv.plan_info(cv.plan_desc(a.layout, p.layout, n), 0))
